# decode step beside the GEMM under sustained load (power cap): short vs long runs, clocks sampled
mkdir -p gpurun_out
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv -lms 200 > gpurun_out/interf_clocks.csv &
SMI=$!
DEC_SMS=74 VARIANTS=none,bn256_gm32 STEPS=6 GEMMS=70 timeout 600 python scripts/interference.py 2>&1 | grep slot_order
DEC_SMS=74 VARIANTS=bn256_gm32 STEPS=80 GEMMS=600 timeout 600 python scripts/interference.py 2>&1 | grep slot_order
kill $SMI
python - <<'P'
import csv
rows=list(csv.reader(open('gpurun_out/interf_clocks.csv')))[1:]
cl=[int(r[1].split()[0]) for r in rows if r[1].strip().split()[0].isdigit()]
pw=[float(r[2].split()[0]) for r in rows if r[2].strip().split()[0].replace('.','').isdigit()]
print('clock MHz min/median/max', min(cl), sorted(cl)[len(cl)//2], max(cl), 'power max', max(pw))
P
