for v in nc ncb nc64; do
 for n in 74; do
  echo "== $v $n"
  timeout 300 env DS_LIB=paper_2603_15042_b200/_var_$v.so NSM=$n python scripts/attn_trace.py 2>&1 | grep nsm | head -1
  timeout 300 env DS_LIB=paper_2603_15042_b200/_var_$v.so NSM=$n LAYERS=8 python scripts/block_stats.py 2>&1 | grep "attn"
 done
done
