# config 4b after the headline legs (the sequence in which it timed out)
mkdir -p gpurun_out
timeout 1200 python bench.py --steps 6 --warmup 3 --no-config13 --no-config5 --no-config4 --no-cpu-baseline > gpurun_out/c4b_seq.json 2> gpurun_out/c4b_seq.err; echo rc=$?
python -c "import json;d=json.loads(open('gpurun_out/c4b_seq.json').read().strip().splitlines()[-1]);print(str(d.get('config4b'))[:800])"
grep -n 'TIMEOUT' -A4 gpurun_out/c4b_seq.err | cut -c1-4000 | head -30
