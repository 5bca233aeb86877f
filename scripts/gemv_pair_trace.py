"""Phases of the two-slab gate_up blocks inside a decode step on the
executor (dbg stamps): start, dependency seen, slab 0 / slab 1 accumulators
final, end; relative to the previous launch's completion."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
nsm = int(os.environ.get("NSM", "74"))
m = DecodeModel(DecodeConfig(layers=4))
names = [r[0] for r in m.records]
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=0)
t = dom.tenant("d", 0)
kids = m.register(dom)
want = {}
for i, (sid, body, grid, args, _) in m.variant_records["gu_pair"].items():
    d = torch.zeros(grid[0] * 8, dtype=torch.int64, device="cuda")
    args.dbg = d.data_ptr()
    want[i] = d
torch.cuda.synchronize()
kp = m.register_variant(dom, kids, "gu_pair")
dom.start()
dom.quota_set(dom.mask(t, 0, nsm))
for _ in range(3):
    for k in kp: last = dom.launch(t, k)
dom.wait(t, last)
cs = dom.poll(1 << 20)[-len(kp):]
for i, d in list(want.items())[1:3]:
    T0 = cs[i - 1].t_end
    rows = d.cpu().view(-1, 8).tolist()
    def rel(j):
        v = [(r[j] - T0) / 1e3 for r in rows if r[j]]
        return [round(statistics.median(v), 1), round(max(v), 1)] if v else None
    print(json.dumps({"nsm": nsm, "blocks": len(rows), "kernel_end": round((cs[i].t_end - T0) / 1e3, 1), "start": rel(0),
                      "dep_seen": rel(7), "slab0_done": rel(1), "slab1_done": rel(2), "epi_done": rel(5), "end": rel(6)}))
dom.stop(); dom.close()
