"""Solo (plain grid) launches of the tenant bodies for ncu.

  python scripts/profile_solo.py gemm        # bf16 GEMM 8192^3 x3
  python scripts/profile_solo.py decode      # one full decode step (163 launches) x2
  python scripts/profile_solo.py gate_up|attn|qkv|lm_head   # that decode kernel x3
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig, TrainGemm
from fractions import Fraction

what = sys.argv[1] if len(sys.argv) > 1 else "gemm"
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=0)
s = torch.cuda.current_stream().cuda_stream
if what == "gemm":
    g = TrainGemm()
    k = g.register(dom)
    for _ in range(3): dom.solo(k, s)
else:
    m = DecodeModel(DecodeConfig(layers=32 if what == "decode" else 1))
    kids = m.register(dom)
    names = [r[0] for r in m.records]
    if what == "decode":
        for _ in range(2):
            for k in kids: dom.solo(k, s)
    else:
        k = kids[names.index("decode/" + what)]
        for _ in range(3): dom.solo(k, s)
torch.cuda.synchronize()
dom.close()
print("done", what)
