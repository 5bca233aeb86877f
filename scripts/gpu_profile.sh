# round profiling: launch list of one decode step (solo plain-grid launches of
# the same bodies: the persistent executor cannot be replayed by ncu) and one
# --set full capture per hot kernel
set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_decode.csv \
    python scripts/profile_solo.py decode > /dev/null 2>&1
for k in attn gate_up lm_head qkv o down; do
  ncu --set full --clock-control none --import-source on -k regex:ds_solo_kernel -s 1 -c 1 \
      -o gpurun_out/prof_$k -f python scripts/profile_solo.py $k > gpurun_out/prof_$k.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:ds_solo_kernel -s 1 -c 1 \
    -o gpurun_out/prof_gemm -f python scripts/profile_solo.py gemm > gpurun_out/prof_gemm.log 2>&1
ls -la gpurun_out/
