for i in 1 2; do
  timeout 1500 python bench.py > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err
  python -c "
import json
d=json.loads(open('gpurun_out/bench_$i.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['train_tflops'], d['timeslice'], d['tpot_distribution_ms']['tpot_first'], d['solo'], d['clocks'], d['bit_exact_vs_solo'], d['roofline']['frac'])
print('c4', json.dumps(d['config4'])[:600])
print('c3', [(r['unit'][:22], r['period_us'], r['yield_us_p50'], r['yield_us_p99'], r['lost_throughput']) for r in d['config3']['sweep']])
"
done
