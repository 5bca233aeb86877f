# fused split-K fold: parity, then the ResNet stream with fused folds for S <= 0 / 8 / 16
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_resnet.py -q 2>&1 | tail -2
for f in 0 8 16 0 8 16; do
  DS_RESNET_FUSE_FOLD=$f timeout 300 python scripts/perf_resnet.py > /dev/null 2>&1
  python -c "import json;d=json.load(open('gpurun_out/perf_resnet.json'));print('fuse<=$f', round(d['iter_ms'],3), round(d['tflops'],1))"
done
