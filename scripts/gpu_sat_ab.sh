# decode saturation tier A/B on one box (headline legs only)
mkdir -p gpurun_out
for sat in 1/2 3/4 1/2 3/4; do
  timeout 900 python bench.py --decode-sat $sat --no-config13 --no-config5 --no-config4 --no-config4b --no-cpu-baseline > gpurun_out/sat.json 2> gpurun_out/sat.err; echo rc=$?
  python -c "
import json;d=json.loads(open('gpurun_out/sat.json').read().strip().splitlines()[-1])
print('sat=$sat', d['value'], d['train_tflops'], d['timeslice']['p99_tpot_ms'], d['timeslice']['train_tflops'], d['bit_exact_vs_solo'], d['clocks']['sm_mhz'], d['tpot_distribution_ms']['tpot_first']['p50'])"
done
