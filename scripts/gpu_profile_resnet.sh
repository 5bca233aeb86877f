mkdir -p gpurun_out
for T in 1 4; do
  DS_RESNET_TILES=$T timeout 300 ncu --set full --clock-control none --import-source on -k regex:ds_solo_kernel -s 2 -c 1 \
    -o gpurun_out/resnet_conv1_fwd_t$T -f python scripts/profile_resnet_gemm.py > gpurun_out/ncu_resnet_t$T.log 2>&1; echo T=$T rc=$?
  ncu -i gpurun_out/resnet_conv1_fwd_t$T.ncu-rep --page raw --csv > gpurun_out/resnet_conv1_fwd_t$T.csv 2>/dev/null
done
