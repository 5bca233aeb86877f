# idle-SM lending on/off under TPOT-First (headline legs only), same box, with clocks / power sampled
mkdir -p gpurun_out
for L in 0 1; do
  nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > gpurun_out/lend_power_$L.csv &
  SMI=$!
  DS_BENCH_LEND=$L timeout 900 python bench.py --steps 10 --no-config13 --no-config5 --no-config4 --no-config4b --no-cpu-baseline > gpurun_out/lend.json 2> gpurun_out/lend_$L.err; echo rc=$?
  kill $SMI
  python -c "
import json;d=json.loads(open('gpurun_out/lend.json').read().strip().splitlines()[-1])
print('lend=$L', 'p99', d['value'], 'train', d['train_tflops'], 'p50', d['tpot_distribution_ms']['tpot_first']['p50'], 'clocks', d['clocks'])"
  python - <<P
import csv, statistics
rows=[r for r in csv.reader(open('gpurun_out/lend_power_$L.csv')) if len(r)>=3]
cl=[float(r[1]) for r in rows]; pw=[float(r[2]) for r in rows]
hi=[(c,p) for c,p in zip(cl,pw) if p>500]
print('lend=$L samples', len(rows), 'loaded', len(hi), 'clock median', statistics.median([c for c,_ in hi]) if hi else None, 'power median', statistics.median([p for _,p in hi]) if hi else None)
P
done
