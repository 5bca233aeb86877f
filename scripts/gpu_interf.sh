# decode step alone vs beside the training GEMM, at 74 / 111 / 148 decode SMs
mkdir -p gpurun_out
for dn in 74 111 148; do
  DEC_SMS=$dn VARIANTS=none,bn256_gm32 STEPS=6 timeout 600 python scripts/interference.py 2>&1 | grep slot_order
done
