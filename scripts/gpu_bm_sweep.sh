for cfg in "|" "qkv:1,o:1|qkv:64,o:64" "qkv:2,o:2|qkv:64,o:64" "qkv:3,o:4|qkv:64,o:64" "down:2|down:64"; do
 sp=${cfg%%|*}; bm=${cfg##*|}
 for n in 74 148; do
   SPLITS=$sp BMS=$bm NSM=$n LAYERS=8 timeout 300 python scripts/critpath.py 2>&1 | grep -v Warn | python -c "
import sys,json
tot=0; out=[]
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        if d['n']>1: tot+=d['incr_us']; out.append(f\"{d['k'][7:]}={d['incr_us']}\")
print('S=[$sp] BM=[$bm] nsm=$n', ' '.join(out), 'layer_us', round(tot,1))
"
 done
done
