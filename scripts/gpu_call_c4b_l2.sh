mkdir -p gpurun_out
timeout 900 python bench.py --only-config4b --steps 2 --warmup 3 --burst-units 30 > gpurun_out/c4b.json 2> gpurun_out/c4b.err; echo c4b=$?
tail -c 1500 gpurun_out/c4b.json; grep -n 'TIMEOUT' -A3 gpurun_out/c4b.err | cut -c1-3000 | head -20
GMS="8 16 32 64" HINTS="0 4 9" bash scripts/gpu_gemm_l2.sh
