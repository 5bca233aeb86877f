"""Per-kernel block statistics of one decode step at a given SM quota:
lane-busy fraction of the kernel's critical span, mean block time, and the
HBM bandwidth a lane sustains while it runs a block."""
import os, sys, json, statistics, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
layers = int(os.environ.get("LAYERS", "8"))
nsm = int(os.environ.get("NSM", "74"))
m = DecodeModel(DecodeConfig(layers=layers, attn_splits=int(os.environ.get("ASPLIT", "1"))),
                split_override=os.environ.get("SPLITS", ""), bm_override=os.environ.get("BMS", ""))
torch.cuda.synchronize()
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=1 << 22)
t = dom.tenant("decode", 0)
kids = m.register(dom)
dom.start()
dom.quota_set(dom.mask(t, 0, nsm))
for _ in range(2):
    for k in kids: last = dom.launch(t, k)
dom.wait(t, last); dom.poll(1 << 16); dom.clear_logs()
s0 = last + 1
for k in kids: last = dom.launch(t, k)
dom.wait(t, last)
cs = dom.poll(1 << 16)
bl = dom.block_log()
by = collections.defaultdict(list)
for b in bl: by[b.seq].append(b)
agg = collections.defaultdict(lambda: collections.defaultdict(float))
prev_end = None
for i, k in enumerate(kids):
    blocks = by[s0 + i]
    c = cs[i]
    start = c.t_first_claim if prev_end is None else max(c.t_first_claim, prev_end)
    span = c.t_end - start
    prev_end = c.t_end
    name, _, grid, _, nbytes = m.records[i]
    a = agg[name]
    a["n"] += 1
    a["span_us"] += span / 1e3
    a["busy_frac"] += sum(min(b.t_end, c.t_end) - max(b.t_start, start) for b in blocks if b.t_end > start) / (2 * nsm * span)
    a["block_us"] += statistics.mean((b.t_end - b.t_start) / 1e3 for b in blocks)
    a["lane_GBps"] += (nbytes / len(blocks)) / statistics.mean(b.t_end - b.t_start for b in blocks)
    a["blocks"] = len(blocks)
    a["GBps"] += nbytes / span
step = (cs[-1].t_end - cs[0].t_first_claim) / 1e3
print("nsm", nsm, "layers", layers, "S", m.S, "step_us", round(step, 1))
for name, a in agg.items():
    n = a["n"]
    print(json.dumps({"k": name, "count": int(n), "blocks": int(a["blocks"]), "span_us": round(a["span_us"] / n, 1),
                      "busy": round(a["busy_frac"] / n, 2), "block_us": round(a["block_us"] / n, 1),
                      "lane_GBps": round(a["lane_GBps"] / n, 1), "GBps": round(a["GBps"] / n, 1)}))
dom.stop(); dom.close()
