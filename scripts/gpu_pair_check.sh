timeout 600 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/t_dec.log 2>&1; echo dec=$?; tail -3 gpurun_out/t_dec.log
for pair in 0 1; do
 for n in 74 148; do
  echo "== pair=$pair nsm=$n"
  DS_GU_PAIR=$pair NSM=$n LAYERS=8 timeout 300 python scripts/critpath.py 2>&1 | grep -v Warn | python -c "
import sys,json
tot=0
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        if d['n']>1: tot+=d['incr_us']; print(d['k'], d['incr_us'], d['nblocks'])
    elif 'step_us' in l: print(l.strip())
print('layer_us', round(tot,1))
"
 done
done
