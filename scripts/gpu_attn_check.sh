timeout 300 python -m pytest tests/test_gpu_attention.py tests/test_gpu_decode.py -x -q > gpurun_out/t_attn.log 2>&1; echo attn=$?; tail -3 gpurun_out/t_attn.log
for n in 74 148; do
 timeout 300 env NSM=$n LAYERS=8 python scripts/block_stats.py 2>&1 | grep "attn\|step_us"
 timeout 200 env DS_LIB=paper_2603_15042_b200/_var_trace.so NSM=$n python scripts/attn_timeline.py 2>&1 | grep nsm | head -1
done
