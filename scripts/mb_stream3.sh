B=scripts/mb_stream
for cfg in "56 2" "74 2" "8 2" "112 1"; do
  set -- $cfg
  $B $1 $2 5 1 0 4 2 16 0
  $B $1 $2 2 1 0 8 2 32 0
  $B $1 $2 4 1 0 4 2 20 0
done
