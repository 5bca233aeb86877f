"""Lane-occupancy timeline of decode kernels inside one step (executor, full GPU)."""
import os, sys, json, statistics, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
layers = int(os.environ.get("LAYERS", "4"))
nsm = int(os.environ.get("NSM", "148"))
m = DecodeModel(DecodeConfig(layers=layers), split_override=os.environ.get("SPLITS", ""))
print("S", m.S)
torch.cuda.synchronize()
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=1 << 22)
t = dom.tenant("decode", 0)
kids = m.register(dom)
dom.start()
dom.quota_set(dom.mask(t, 0, nsm))
for _ in range(3):
    for k in kids: last = dom.launch(t, k)
dom.wait(t, last); dom.poll(1 << 16); dom.clear_logs()
s0 = last + 1
for k in kids: last = dom.launch(t, k)
dom.wait(t, last)
cs = dom.poll(1 << 16)
bl = dom.block_log()
lanes = 2 * nsm
byk = collections.defaultdict(list)
for b in bl: byk[b.seq].append(b)
T0 = min(b.t_start for b in bl)
agg = collections.defaultdict(lambda: [0, 0, 0, 0])
rows = []
for i, k in enumerate(kids):
    seq = s0 + i
    blocks = byk[seq]
    st = min(b.t_start for b in blocks); en = max(b.t_end for b in blocks)
    busy = sum(b.t_end - b.t_start for b in blocks)
    name = m.records[i][0]
    a = agg[name]; a[0] += en - st; a[1] += busy; a[2] += 1; a[3] += m.records[i][4]
    if i < 12: rows.append((name, round((st - T0) / 1e3, 1), round((en - T0) / 1e3, 1), round(busy / (lanes * (en - st)), 2), len(blocks)))
for r in rows: print(r)
tot_span = (max(b.t_end for b in bl) - T0) / 1e3
print("step_us", round(tot_span, 1))
for name, a in agg.items():
    print(json.dumps({"k": name, "span_us_avg": round(a[0] / a[2] / 1e3, 1), "occupancy": round(a[1] / (lanes * a[0]), 2),
                      "GBps_span": round(a[3] / (a[0] / a[2]) , 1) if a[0] else 0, "count": a[2]}))
dom.stop(); dom.close()
