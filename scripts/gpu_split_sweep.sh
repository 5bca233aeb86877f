for sp in "" "qkv:2" "qkv:4" "o:2" "o:3" "down:3" "down:6" "qkv:2,o:2,down:3"; do
 for n in 74 148; do
   echo "== S=$sp nsm=$n"
   SPLITS=$sp NSM=$n LAYERS=8 timeout 300 python scripts/critpath.py 2>&1 | grep -v Warn | python -c "
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
