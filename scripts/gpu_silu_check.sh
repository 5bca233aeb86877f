mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_decode.py -q -x 2>&1 | tail -1
KERNELS=gate_up timeout 300 python scripts/gemv_solo_trace.py
for i in 1 2; do
  echo "critpath nsm=148: $(NSM=148 LAYERS=8 timeout 300 python scripts/critpath.py 2>&1 | grep step_us)"
  echo "critpath nsm=74: $(NSM=74 LAYERS=8 timeout 300 python scripts/critpath.py 2>&1 | grep step_us)"
done
timeout 300 python scripts/gemv_pf_solo.py 2>&1 | tail -1
