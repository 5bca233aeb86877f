# tune the ResNet stream's split-K GEMMs, then the stream with and without the table
mkdir -p gpurun_out
timeout 1200 python scripts/autotune_resnet.py > gpurun_out/autotune.log 2>&1; echo tune=$?; tail -3 gpurun_out/autotune.log
for tu in 0 1 0 1; do
  DS_RESNET_TUNED=$tu timeout 300 python scripts/perf_resnet.py > /dev/null 2>&1
  python -c "import json;d=json.load(open('gpurun_out/perf_resnet.json'));print('tuned=$tu', round(d['iter_ms'],3), round(d['tflops'],1))"
done
timeout 300 python -m pytest tests/test_gpu_gemm.py -q 2>&1 | tail -1
