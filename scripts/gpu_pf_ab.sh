# co-located A/B of the early-start L2 prefetch depth (config 2 only)
for i in 1 2; do
for pf in "" "qkv:0,attn:0,o:0,gu:0,down:0,lm:0" "qkv:256,attn:256,o:256,gu:256,down:256,lm:0"; do
  DS_L2PF=$pf timeout 900 python bench.py --no-config13 --no-config5 --no-config4 --no-config4b --no-cpu-baseline > gpurun_out/b_pf.json 2> gpurun_out/b_pf.err
  python -c "
import json
d=json.loads(open('gpurun_out/b_pf.json').read().strip().splitlines()[-1])
print('pf=[$pf]', d['value'], d['tpot_distribution_ms']['tpot_first']['p50'], d['train_tflops'], d['solo']['decode_step_ms'], d['clocks']['sm_mhz'])
"
done
done
