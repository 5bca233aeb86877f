"""Where the time goes after a decode GEMV's dependency resolves (inside a
real decode step on the executor): per-block phase stamps relative to the
previous launch's completion T0."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
nsm = int(os.environ.get("NSM", "148"))
m = DecodeModel(DecodeConfig(layers=4))
names = [r[0] for r in m.records]
want = {}  # record index -> dbg tensor
layer2 = [i for i, n in enumerate(names) if n.startswith("decode/")][2 + 5 * 2: 2 + 5 * 3]  # layer 2's 5 launches
for i in layer2:
    sid, body, grid, args, _ = m.records[i]
    if body == _abi.BODY_GEMV_BF16:
        d = torch.zeros(grid[0] * 8, dtype=torch.int64, device="cuda")
        args.dbg = d.data_ptr()
        want[i] = d
torch.cuda.synchronize()
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=0)
t = dom.tenant("d", 0)
kids = m.register(dom)
dom.start()
dom.quota_set(dom.mask(t, 0, nsm))
for _ in range(3):
    for k in kids: last = dom.launch(t, k)
dom.wait(t, last)
cs = dom.poll(1 << 20)[-len(kids):]
mask = (1 << 63) - 1
for i, d in want.items():
    T0 = cs[i - 1].t_end
    rows = d.cpu().view(-1, 8).tolist()
    def rel(j, sel=lambda r: True):
        v = [((r[j] & mask) - T0) / 1e3 for r in rows if sel(r) and (r[j] & mask)]
        return [round(statistics.median(v), 1), round(max(v), 1)] if v else None
    comb = lambda r: (r[2] >> 63) & 1
    print(json.dumps({"k": names[i], "blocks": len(rows), "end": round((cs[i].t_end - T0) / 1e3, 1),
                      "start": rel(0), "dep_seen(7)": rel(7), "main_end(1)": rel(1),
                      "comb_got(2)": rel(2, comb), "comb_sum(3)": rel(3, comb), "stats(4)": rel(4, comb),
                      "store(5)": rel(5, comb), "end(6)": rel(6)}), flush=True)
dom.stop(); dom.close()
