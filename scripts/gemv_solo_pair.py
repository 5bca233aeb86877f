"""gate_up one-slab vs two-slab records as plain-grid solo launches (CUDA
events): the body's own streaming rate without the executor."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
m = DecodeModel(DecodeConfig(layers=2))
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=0)
kids = m.register(dom)
kp = m.register_variant(dom, kids, "gu_pair")
names = [r[0] for r in m.records]
i = names.index("decode/gate_up")
s = torch.cuda.current_stream()
for label, k in (("one-slab 224 blocks", kids[i]), ("two-slab 112 blocks", kp[i])):
    for _ in range(3): dom.solo(k, s.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10): dom.solo(k, s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 10
    print(json.dumps({"gate_up": label, "solo_us": round(us, 1), "GBps": round(m.records[i][4] / us / 1e3, 1)}))
dom.close()
