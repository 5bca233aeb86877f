B=scripts/mb_stream
for nsm in 74 148; do
  $B $nsm 2 5 1 0 4 2 16 0
  $B $nsm 2 5 1 0 4 2 16 1
  $B $nsm 2 5 1 0 4 8 16 0
  $B $nsm 2 5 1 0 4 8 16 1
done
