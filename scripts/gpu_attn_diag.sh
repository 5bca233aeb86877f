for v in nc ldsm; do
  echo "== $v"
  timeout 300 env DS_LIB=paper_2603_15042_b200/_var_$v.so NSM=74 python scripts/attn_trace.py 2>&1 | grep nsm | head -1
  timeout 300 env DS_LIB=paper_2603_15042_b200/_var_$v.so NSM=74 LAYERS=8 python scripts/block_stats.py 2>&1 | grep "attn"
done
