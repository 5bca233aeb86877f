# ResNet stream A/B: split-K tile width (narrow vs wide) x multi-tile blocks
mkdir -p gpurun_out
for cfg in "0 8" "1 8" "1 1" "0 8" "1 8"; do set -- $cfg
  DS_RESNET_WIDE=$1 DS_RESNET_TILES=$2 timeout 300 python scripts/perf_resnet.py > gpurun_out/perf_resnet_w$1_t$2.log 2>&1; echo rc=$?
  python -c "import json;d=json.load(open('gpurun_out/perf_resnet.json'));print('wide=$1 tiles=$2', round(d['iter_ms'],3), round(d['tflops'],1))"
  cp gpurun_out/perf_resnet.json gpurun_out/perf_resnet_w$1_t$2.json
done
