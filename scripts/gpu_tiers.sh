for t in "1/4,1/2,3/4,1" "1/4,1/2,1" "1/4,3/4,1"; do
  tag=$(echo $t | tr '/,' '_-')
  timeout 300 python bench.py --steps 20 --tiers $t --no-cpu-baseline > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$tag.json'));print('$t', d['value'], d['train_tflops'], d['timeslice'], d['e2e']['value'], d['bit_exact_vs_solo'])"
done
