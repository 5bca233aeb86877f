for v in default k3v3 k4v2 nocomp; do
  for n in 74 148; do
    if [ $v = default ]; then L=""; else L=paper_2603_15042_b200/_var_$v.so; fi
    echo "== $v nsm=$n"
    DS_LIB=$L NSM=$n LAYERS=8 python scripts/block_stats.py 2>&1 | grep -v Warn | grep "attn\|step_us"
  done
done
echo "== asplit2 nsm=74"; ASPLIT=2 NSM=74 LAYERS=8 python scripts/block_stats.py 2>&1 | grep "attn\|step_us"
