# co-located A/B of the decode tier's bit-identical variants (config 2 only)
for i in 1 2; do
for hv in 0 gu_pair lm_multi gu_pair,lm_multi; do
  DS_HALF_VARIANTS=$hv timeout 900 python bench.py --no-config13 --no-config5 --no-config4 --no-config4b --no-cpu-baseline > gpurun_out/b_hv.json 2> gpurun_out/b_hv.err
  python -c "
import json
d=json.loads(open('gpurun_out/b_hv.json').read().strip().splitlines()[-1])
print('half_variants=$hv', d['value'], d['tpot_distribution_ms']['tpot_first']['p50'], d['train_tflops'], d['bit_exact_vs_solo'], d['clocks']['sm_mhz'])
"
done
done
