# sliding L2 prefetch distance for the decode GEMVs: solo kernels, then the decode step on the executor
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_decode.py -q -x 2>&1 | tail -1
for d in 0 4 8 16 0 8; do DS_GEMV_PF_AHEAD=$d timeout 300 python scripts/gemv_pf_solo.py 2>&1 | tail -1; done
for d in 0 8 0 8; do
  echo "critpath pf=$d nsm=148: $(DS_GEMV_PF_AHEAD=$d NSM=148 LAYERS=8 timeout 300 python scripts/critpath.py 2>&1 | grep step_us)"
  echo "critpath pf=$d nsm=74: $(DS_GEMV_PF_AHEAD=$d NSM=74 LAYERS=8 timeout 300 python scripts/critpath.py 2>&1 | grep step_us)"
done
