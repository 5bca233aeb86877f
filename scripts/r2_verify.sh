set -x
timeout 600 python -m pytest tests/test_gpu_boundary.py -q -s > gpurun_out/pytest_boundary.log 2>&1; echo boundary=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_boundary.log; tail -5 gpurun_out/pytest_gpu.log
