# split-K fold row grouping A/B on the ResNet stream + the new parity tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/pytest_gemm.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gemm.log
for f in 0 1 0 1; do
  DS_RESNET_FOLD_WIDE=$f timeout 300 python scripts/perf_resnet.py > gpurun_out/perf_resnet_f$f.log 2>&1; echo rc=$?
  python -c "import json;d=json.load(open('gpurun_out/perf_resnet.json'));print('fold_wide=$f', round(d['iter_ms'],3), round(d['tflops'],1), round(sum(r[1] for r in d['by_excess_us'] if r[0].endswith('/fold')),1))"
  cp gpurun_out/perf_resnet.json gpurun_out/perf_resnet_f$f.json
done
