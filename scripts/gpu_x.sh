timeout 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -1
DS_LIB=paper_2603_15042_b200/_var_trace.so NSM=74 timeout 200 python scripts/attn_timeline_tc.py > gpurun_out/tl_tc.txt 2>&1
for tcv in 0 1; do for n in 74 148; do
   echo "== tc=$tcv nsm=$n"
   DS_ATTN_TC=$tcv NSM=$n LAYERS=8 timeout 300 python scripts/critpath.py 2>&1 | grep attn | cut -c1-80
done; done
