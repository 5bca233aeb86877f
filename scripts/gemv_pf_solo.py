"""Decode projections as plain-grid solo launches (the bench roofline's
setting), events-timed, for the current DS_GEMV_PF_AHEAD: us and GB/s per
kernel.  Each launch streams a different layer's weights (cold L2)."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
m = DecodeModel(DecodeConfig(layers=8))
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=0)
kids = m.register(dom)
names = [r[0] for r in m.records]
s = torch.cuda.current_stream()
out = {"pf_ahead": int(os.environ.get("DS_GEMV_PF_AHEAD", "0"))}
for k in ("qkv", "o", "gate_up", "down"):
    idx = [i for i, n in enumerate(names) if n == "decode/" + k]
    for i in idx: dom.solo(kids[i], s.cuda_stream)
    torch.cuda.synchronize()
    ts = []
    for rep in range(3):
        for i in idx:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); dom.solo(kids[i], s.cuda_stream); e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
    us = statistics.median(ts)
    out[k] = {"us": round(us, 2), "GBps": round(m.records[idx[0]][4] / (us * 1e3), 1)}
print(json.dumps(out))
dom.close()
