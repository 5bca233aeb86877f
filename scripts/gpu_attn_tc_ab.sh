DS_ATTN_TC=1 timeout 600 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/t_dec_tc.log 2>&1; echo dec_tc=$?; tail -2 gpurun_out/t_dec_tc.log
for i in 1 2; do
for tcv in 0 1; do
 for n in 74 148; do
   echo "== tc=$tcv nsm=$n"
   DS_ATTN_TC=$tcv NSM=$n LAYERS=8 timeout 300 python scripts/critpath.py 2>&1 | grep -v Warn | python -c "
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
done
