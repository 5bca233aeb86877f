"""lm_head GEMV block phases at an SM quota: mainloop streaming rate vs
block overheads (dbg[0] start, dbg[7] dep satisfied, dbg[1] mainloop end,
dbg[6] body end)."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
from fractions import Fraction
nsm = int(os.environ.get("NSM", "37"))
m = DecodeModel(DecodeConfig(layers=1))
names = [r[0] for r in m.records]
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=0)
t = dom.tenant("d", 0)
i = names.index("decode/lm_head")
sid, body, grid, args, nbytes = m.records[i]
dbg = torch.zeros(grid[0] * 8, dtype=torch.int64, device="cuda")
args.dbg = dbg.data_ptr()
kid = dom.kernel(sid, body, grid, args)
torch.cuda.synchronize()
dom.start()
dom.quota_set(dom.mask(t, 0, nsm))
for _ in range(3): last = dom.launch(t, kid)
dom.wait(t, last)
d = dbg.cpu().view(grid[0], 8).tolist()
mask = (1 << 63) - 1
main = [((r[1] & mask) - max(r[0], r[7])) / 1e3 for r in d]
tot = [((r[6] & mask) - r[0]) / 1e3 for r in d]
per_block = nbytes / grid[0]
def ph(rows, a, b):
    v = [((r[b] & mask) - (r[a] & mask)) / 1e3 for r in rows if (r[b] & mask) and (r[a] & mask)]
    return round(statistics.median(v), 2) if v else None
last = [r for r in d if (r[2] >> 63) & 1]
other = [r for r in d if not ((r[2] >> 63) & 1)]
print(json.dumps({"other": {"pre": ph(other, 0, 7), "main": ph(other, 7, 1), "ticket": ph(other, 1, 2),
                            "to_end": ph(other, 2, 6)},
                  "last": {"pre": ph(last, 0, 7), "main": ph(last, 7, 1), "ticket": ph(last, 1, 2),
                           "combine": ph(last, 2, 3), "stats": ph(last, 3, 4), "store": ph(last, 4, 5),
                           "teardown": ph(last, 5, 6)}}))
print(json.dumps({"nsm": nsm, "blocks": grid[0], "KB_per_block": per_block / 1024,
                  "main_us_med": round(statistics.median(main), 2), "body_us_med": round(statistics.median(tot), 2),
                  "main_GBps_lane": round(per_block / statistics.median(main) / 1e3, 1)}), flush=True)
dom.stop(); dom.close()
