# three default bench runs back to back: run-to-run spread of the headline line
for i in 1 2 3; do
  timeout 1500 python bench.py > gpurun_out/bench_r$i.json 2> gpurun_out/bench_r$i.err
  python -c "
import json
d=json.loads(open('gpurun_out/bench_r$i.json').read().strip().splitlines()[-1])
print(json.dumps({'run': $i, 'p99_tpot_ms': d['value'], 'p50': d['tpot_distribution_ms']['tpot_first']['p50'], 'e2e': d['e2e']['value'],
  'train_tflops': d['train_tflops'], 'timeslice_p99': d['timeslice']['p99_tpot_ms'], 'timeslice_tflops': d['timeslice']['train_tflops'],
  'solo_step_ms': d['solo']['decode_step_ms'], 'sm_mhz': d['clocks']['sm_mhz'], 'bit_exact': d['bit_exact_vs_solo'],
  'roofline_frac': d['roofline']['frac'], 'c4_tpot_first': d['config4']['tpot_first']['p99_tpot_ms'], 'c4_temporal': d['config4']['temporal']['p99_tpot_ms']}))
"
done
