"""Per-chunk timeline of the tcgen05 attention (DS_ATTN_TRACE build, DS_ATTN_TC=1):
softmax stream 0 (top, S landed, P written, p_ready) and the MMA thread's QK / PV issue times."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["DS_ATTN_TC"] = "1"
import torch
from fractions import Fraction
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
nsm = int(os.environ.get("NSM", "74"))
m = DecodeModel(DecodeConfig(layers=4))
names = [r[0] for r in m.records]
want = {}
for i, n in enumerate(names):
    if n == "decode/attn":
        _, _, grid, args, _ = m.records[i]
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
i, d = list(want.items())[2]
rows = d.cpu().view(-1, 128).tolist()
for bidx in (0, 200):
    r = rows[bidx]
    t0 = r[7]
    rel = lambda x: round((x - t0) / 1e3, 2) if x else None
    its = [{"ci": c, "qk": rel(r[80 + c]), "top": rel(r[8 + 4 * c]), "S": rel(r[9 + 4 * c]), "P": rel(r[10 + 4 * c]),
            "ready": rel(r[11 + 4 * c]), "pv": rel(r[64 + c])} for c in range(14)]
    print(json.dumps({"nsm": nsm, "block": bidx, "start": rel(r[0]), "end": rel(r[6]), "iters": its}))
dom.stop(); dom.close()
