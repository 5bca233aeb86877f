"""GEMV phase timestamps inside a real decode step (early start active)."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
m = DecodeModel(DecodeConfig(layers=2))
names = [r[0] for r in m.records]
dbgs = {}
for name in ("decode/qkv", "decode/o", "decode/gate_up", "decode/down"):
    i = names.index(name, names.index("decode/embed") + 6)  # layer 1 instance
    sid, body, grid, args, _ = m.records[i]
    dbg = torch.zeros(grid[0] * 8, dtype=torch.int64, device="cuda")
    args.dbg = dbg.data_ptr()
    dbgs[name] = (dbg, grid[0], i)
torch.cuda.synchronize()
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=0)
t = dom.tenant("d", 0)
kids = m.register(dom)
dom.start(); dom.quota_set(dom.mask(t, 0, dom.num_sms))
for _ in range(3):
    for k in kids: last = dom.launch(t, k)
dom.wait(t, last)
for name, (dbg, g, i) in dbgs.items():
    d = dbg.cpu().view(g, 8).tolist()
    mask = (1 << 63) - 1
    T = min(r[0] for r in d)
    dep = [((r[7] & mask) - T) / 1e3 for r in d]
    last = [r for r in d if (r[2] >> 63) & 1]
    def med(rows, a, b):
        v = [((r[b] & mask) - (r[a] & mask)) / 1e3 for r in rows]; return [round(statistics.median(v), 2), round(max(v), 2)]
    print(json.dumps({"k": name, "blocks": g, "start_spread": round((max(r[0] for r in d) - T) / 1e3, 1),
        "dep_resolved(min,med,max)": [round(min(dep), 1), round(statistics.median(dep), 1), round(max(dep), 1)],
        "dep->mainloop_end": med(d, 7, 1), "tick": med(d, 1, 2), "last: comb, norm, mode, tear": [med(last, 2, 3), med(last, 3, 4), med(last, 4, 5), med(last, 5, 6)],
        "end(max) rel": round((max(r[6] for r in d) - T) / 1e3, 1)}))
dom.stop(); dom.close()
