for i in 1 2; do
for p in 0 1; do
  DS_GU_PAIR=$p timeout 1200 python bench.py > gpurun_out/bench_p$p.json 2> gpurun_out/bench_p$p.err
  python -c "
import json
d=json.loads(open('gpurun_out/bench_p$p.json').read().strip().splitlines()[-1])
print('pair=$p', d['value'], d['train_tflops'], d['timeslice']['p99_tpot_ms'], d['timeslice']['train_tflops'], d['solo']['decode_step_ms'], d['clocks']['sm_mhz'], d['bit_exact_vs_solo'])
"
done
done
