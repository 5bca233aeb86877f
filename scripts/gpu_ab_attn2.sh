timeout 300 python -m pytest tests/test_gpu_attention.py tests/test_gpu_decode.py -x -q 2>&1 | tail -1
for i in 1 2 3; do
for v in current prev; do
  if [ $v = current ]; then unset DS_LIB; else export DS_LIB=paper_2603_15042_b200/_var_$v.so; fi
  for n in 74 148; do
   echo "$v nsm=$n $(NSM=$n LAYERS=8 timeout 300 python scripts/critpath.py 2>&1 | grep attn | cut -c1-60)"
  done
done
done
unset DS_LIB
