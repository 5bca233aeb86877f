timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in "" "gu_pair" "gu_pair,lm_multi"; do
 for n in 74 148; do
   echo "V=[$v] nsm=$n $(VARIANTS=$v NSM=$n LAYERS=8 timeout 300 python scripts/critpath.py 2>&1 | grep -E 'lm_head|gate_up' | cut -c1-70 | tr '\n' ' ')"
 done
done
