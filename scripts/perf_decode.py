"""Decode step: plain-stream solo launches vs the coroutine executor (full GPU)."""
import os, sys, json, time, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
layers = int(os.environ.get("LAYERS", "32"))
m = DecodeModel(DecodeConfig(layers=layers))
torch.cuda.synchronize()
print("S", m.S, "step_bytes GB", m.step_bytes / 1e9, flush=True)
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=1 << 22)
t = dom.tenant("decode", _abi.LATENCY_CRITICAL)
kids = m.register(dom)
# solo: the same registered records as plain kernels on one stream
s = torch.cuda.current_stream().cuda_stream
for i in range(2):
    for k in kids: dom.solo(k, s)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
n = 5
e0.record()
for i in range(n):
    for k in kids: dom.solo(k, s)
e1.record(); torch.cuda.synchronize()
solo_ms = e0.elapsed_time(e1) / n
print(json.dumps({"solo_step_ms": solo_ms, "solo_GBps": m.step_bytes / (solo_ms * 1e-3) / 1e9}), flush=True)
dom.start()
dom.quota_set(dom.mask(t, 0, dom.num_sms))
for i in range(2):
    for k in kids: last = dom.launch(t, k)
dom.wait(t, last); dom.poll(); dom.clear_logs()
steps = 5
for i in range(steps):
    for k in kids: last = dom.launch(t, k)
dom.wait(t, last)
cs = dom.poll(100000)
ends = [c.t_end for c in cs]
per_step = [(ends[(i + 1) * len(kids) - 1] - ends[i * len(kids) - 1]) / 1e6 for i in range(1, steps)]
by = collections.defaultdict(list)
for i, c in enumerate(cs):
    rec = m.records[i % len(kids)]
    by[rec[0]].append(((c.t_end - c.t_first_claim) / 1e3, rec[4]))
summary = {k: {"us": sum(x for x, _ in v) / len(v), "GBps": sum(b for _, b in v) / sum(x for x, _ in v) / 1e3} for k, v in by.items()}
gaps = [(cs[i].t_first_claim - cs[i - 1].t_end) / 1e3 for i in range(1, len(cs))]
print(json.dumps({"exec_step_ms": per_step, "exec_GBps": m.step_bytes / (min(per_step) * 1e-3) / 1e9,
                  "kernels": summary, "gap_us_mean": sum(gaps) / len(gaps)}), flush=True)
bl = dom.block_log()
dur = collections.defaultdict(list)
for b in bl:
    dur[m.records[b.seq % len(kids)][0]].append((b.t_end - b.t_start) / 1e3)
print(json.dumps({k: {"blocks": len(v), "mean_us": sum(v)/len(v), "max_us": max(v)} for k, v in dur.items()}), flush=True)
dom.stop(); dom.close()
