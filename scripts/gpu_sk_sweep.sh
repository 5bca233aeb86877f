timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_attention.py -x -q > gpurun_out/t_dec.log 2>&1; echo dec=$?; tail -3 gpurun_out/t_dec.log
for g in "" "gu:296" "gu:296,down:296" "gu:296,down:296,qkv:296,o:296" "gu:296,down:148,qkv:148,o:148" "gu:444,down:296,qkv:296,o:296"; do
 for n in 74 148; do
  echo "== G=$g nsm=$n"
  DS_GEMV_G=$g NSM=$n LAYERS=8 timeout 300 python scripts/critpath.py 2>&1 | grep -v Warn | python -c "
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
