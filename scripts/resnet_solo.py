"""ResNet-50 stream GEMMs as plain-grid solo launches (CUDA events) next to
their executor times: where the per-tile cost comes from."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import ResNetStream
rs = ResNetStream()
names = [r[0] for r in rs.records]
pick = [n for n in names if n in ("resnet/conv1/fwd", "resnet/conv1/wgrad", "resnet/s2b2_3x3/fwd", "resnet/s2b1_3x3/dgrad",
                                   "resnet/s3b0_3x3/dgrad", "resnet/s4b0_3x3/dgrad", "resnet/s1b0_3x3/fwd")]
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=0)
kids = rs.register(dom)
s = torch.cuda.current_stream()
for n in pick:
    i = names.index(n)
    k = kids[i]
    plan = rs.plans[[r[0] for r in rs.records if not r[0].endswith("/fold")].index(n)]
    for _ in range(2): dom.solo(k, s.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(5): dom.solo(k, s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 5
    fl = rs.records[i][4]
    print(json.dumps({"gemm": n, "plan(Mp,Np,Kp,bn,splits)": plan, "grid": rs.records[i][2], "solo_us": round(us, 1),
                      "tflops": round(fl / (us * 1e-6) / 1e12, 1)}), flush=True)
dom.close()
