# A/B of the product library against an experiment build (DS_LIB) inside one call
V=${V:-prev}
for i in 1 2; do
 for lib in "" paper_2603_15042_b200/_var_$V.so; do
  for n in 74 148; do
   echo "== lib=${lib:-current} nsm=$n"
   if [ -n "$lib" ]; then export DS_LIB=$lib; else unset DS_LIB; fi
   NSM=$n LAYERS=8 timeout 300 python scripts/critpath.py 2>&1 | grep -v Warn | python -c "
import sys,json
tot=0
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        if d['n']>1: tot+=d['incr_us']; print(d['k'], d['incr_us'])
print('layer_us', round(tot,1))
"
  done
 done
done
unset DS_LIB
