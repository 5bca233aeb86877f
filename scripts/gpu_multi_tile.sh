# multi-tile GEMM blocks: parity tests, then the ResNet stream A/B (one-tile vs multi-tile records)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -k multi > gpurun_out/pytest_multi.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_multi.log
for T in 1 8 4 1 8; do
  DS_RESNET_TILES=$T timeout 300 python scripts/perf_resnet.py > gpurun_out/perf_resnet_t$T.log 2>&1; echo T=$T rc=$?
  python -c "import json;d=json.load(open('gpurun_out/perf_resnet.json'));print('T=$T', round(d['iter_ms'],3), round(d['tflops'],1))"
  cp gpurun_out/perf_resnet.json gpurun_out/perf_resnet_t$T.json
done
