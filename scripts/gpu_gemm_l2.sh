# GEMM 8192^3 DRAM traffic / speed vs raster group and L2 hints (one gpurun call)
mkdir -p gpurun_out
out=gpurun_out/gemm_l2.jsonl; : > $out
for gm in ${GMS:-8 16 24 32 64}; do for h in ${HINTS:-0 4 15 9 10}; do
  GM=$gm HINT=$h timeout 120 python scripts/gemm_l2_sweep.py >> $out 2>>gpurun_out/gemm_l2.err
  GM=$gm HINT=$h NCU=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
     --clock-control none -k regex:ds_solo_kernel -s 2 -c 1 --csv python scripts/gemm_l2_sweep.py 2>/dev/null \
     | grep -E 'dram__|gpu__time|tensor' | awk -v gm=$gm -v h=$h -F'","' '{print "ncu gm="gm" hint="h" "$(NF-2)" "$NF}' >> gpurun_out/gemm_l2_ncu.txt
done; done
cat $out; cat gpurun_out/gemm_l2_ncu.txt
