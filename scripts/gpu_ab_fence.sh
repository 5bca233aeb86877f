for i in 1 2; do
for lib in "" paper_2603_15042_b200/_var_nofence.so; do
  if [ -n "$lib" ]; then export DS_LIB=$lib; else unset DS_LIB; fi
  echo "== lib=${lib:-current}"
  timeout 300 python scripts/perf_resnet.py 2>&1 | grep -E '"iter_ms"'
  NSM=74 LAYERS=8 timeout 300 python scripts/critpath.py 2>&1 | grep -v Warn | python -c "
import sys,json
tot=0; out=[]
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        if d['n']>1: tot+=d['incr_us']; out.append(f\"{d['k'][7:]}={d['incr_us']}\")
print(' '.join(out), 'layer_us', round(tot,1))
"
done
done
unset DS_LIB
