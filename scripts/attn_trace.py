"""Attention phase breakdown inside a decode step: per block, the prologue
(start -> past wait_prev), the main loop and the merge epilogue (dbg stamps
of bodies/decode.cuh body_attn_decode)."""
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
for i, d in list(want.items())[1:3]:
    rows = d.cpu().view(-1, 8).tolist()
    med = lambda f: round(statistics.median(f(r) for r in rows) / 1e3, 2)
    print(json.dumps({"nsm": nsm, "blocks": len(rows), "prologue_us": med(lambda r: r[7] - r[0]),
                      "main_us": med(lambda r: r[1] - r[7]), "epi_us": med(lambda r: r[6] - r[1])}), flush=True)
dom.stop(); dom.close()
