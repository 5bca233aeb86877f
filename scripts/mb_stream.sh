# sweep of the streaming microbenchmark (scripts/mb_stream.cu)
B=scripts/mb_stream
for nsm in 8 74 148; do
  for mma in 0 1; do
    $B $nsm 2 5 $mma 0 4 2
    $B $nsm 1 5 $mma 0 4 2
    $B $nsm 1 10 $mma 0 4 2
  done
  $B $nsm 2 5 1 128 4 2
  $B $nsm 2 5 1 512 4 2
  $B $nsm 2 5 0 512 4 2
  $B $nsm 2 6 0 0 0 2
  $B $nsm 2 3 1 0 4 2 32
  $B $nsm 2 10 1 0 4 2 8
done
