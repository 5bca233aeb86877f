"""Per-chunk timeline of one attention block inside a decode step (build with
DS_ATTN_TRACE, select with DS_LIB): for warp 0, when each of its chunks was
issued, when it waited for the issue / the data, and when its compute ended."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
nsm = int(os.environ.get("NSM", "74"))
m = DecodeModel(DecodeConfig(layers=4))
names = [r[0] for r in m.records]
want = {}
for i, n in enumerate(names):
    if n == "decode/attn":
        sid, body, grid, args, _ = m.records[i]
        d = torch.zeros(grid[0] * 128, dtype=torch.int64, device="cuda")
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
chunk = _abi.attn_chunk()
groups = 8 // (chunk // 16)
i, d = list(want.items())[2]
rows = d.cpu().view(-1, 128).tolist()
for bidx in (0, 100, 200):
    r = rows[bidx]
    t0 = r[7]
    rel = lambda x: round((x - t0) / 1e3, 2) if x else None
    its = []
    for j in range(12):
        a, b_, c_, e = r[8 + 4 * j: 12 + 4 * j]
        if not a: break
        ci = j * groups
        its.append({"ci": ci, "issued": rel(r[64 + ci]) if ci < 64 else None, "top": rel(a), "spun_to": rel(b_),
                    "landed": rel(c_), "done": rel(e)})
    print(json.dumps({"nsm": nsm, "block": bidx, "start": rel(r[0]), "main_end": rel(r[1]), "end": rel(r[6]),
                      "iters": its}), flush=True)
dom.stop(); dom.close()
