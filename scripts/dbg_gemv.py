"""Phase timestamps inside decode GEMV blocks (solo launch, full GPU)."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, ctypes
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import solo_launch, Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
from fractions import Fraction
m = DecodeModel(DecodeConfig(layers=2))
names = [r[0] for r in m.records]
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=1 << 20)
t = dom.tenant("d", 0)
out = {}
dbgs = {}
for name in ("decode/qkv", "decode/o", "decode/down"):
    i = names.index(name)
    sid, body, grid, args, _ = m.records[i]
    dbg = torch.zeros(grid[0] * 8, dtype=torch.int64, device="cuda")
    args.dbg = dbg.data_ptr()
    dbgs[name] = (dom.kernel(sid, body, grid, args), dbg, grid[0])
torch.cuda.synchronize()
dom.start()
dom.quota_set(dom.mask(t, 0, int(os.environ.get("NSM", "148"))))
for name, (kid, dbg, g) in dbgs.items():
    for _ in range(3): last = dom.launch(t, kid)
    dom.wait(t, last)
    d = dbg.cpu().view(g, 8).tolist()
    t0 = min(r[0] for r in d)
    last_blocks = [r for r in d if (r[2] >> 63) & 1]
    other = [r for r in d if not ((r[2] >> 63) & 1)]
    if not other:
        other = last_blocks
    def ph(rows, a, b, mask=False):
        v = [((r[b] & ((1 << 63) - 1)) - (r[a] & ((1 << 63) - 1))) / 1e3 for r in rows]
        return [round(statistics.median(v), 2), round(max(v), 2)]
    print(json.dumps({"kernel": name, "n_last": len(last_blocks), "n_other": len(other),
        "other: main, tick, end": [ph(other, 0, 1), ph(other, 1, 2), ph(other, 0, 6)],
        "last: main, tick, comb, norm, mode, teardown": [ph(last_blocks, 0, 1), ph(last_blocks, 1, 2), ph(last_blocks, 2, 3), ph(last_blocks, 3, 4), ph(last_blocks, 4, 5), ph(last_blocks, 5, 6)],
        "start spread": round((max(r[0] for r in d) - t0) / 1e3, 2)}), flush=True)
dom.stop(); dom.close()
