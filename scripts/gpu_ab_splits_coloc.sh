# co-located A/B of the GEMV split-K factors (config 2 only)
for i in 1 2; do
for sp in "" "down:5" "down:3" "o:3" "qkv:4" "o:5"; do
  DS_SPLITS=$sp timeout 900 python bench.py --no-config13 --no-config5 --no-config4 --no-config4b --no-cpu-baseline > gpurun_out/b_sp.json 2> gpurun_out/b_sp.err
  python -c "
import json
d=json.loads(open('gpurun_out/b_sp.json').read().strip().splitlines()[-1])
print('splits=[$sp]', d['value'], d['tpot_distribution_ms']['tpot_first']['p50'], d['train_tflops'], d['bit_exact_vs_solo'], d['clocks']['sm_mhz'])
"
done
done
