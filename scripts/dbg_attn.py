import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
m = DecodeModel(DecodeConfig(layers=1))
i = [r[0] for r in m.records].index("decode/attn")
sid, body, grid, args, _ = m.records[i]
dbg = torch.zeros(grid[0] * 8, dtype=torch.int64, device="cuda")
args.dbg = dbg.data_ptr()
torch.cuda.synchronize()
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=0)
t = dom.tenant("d", 0)
k = dom.kernel(sid, body, grid, args)
dom.start(); dom.quota_set(dom.mask(t, 0, dom.num_sms))
for _ in range(3): last = dom.launch(t, k)
dom.wait(t, last)
d = dbg.cpu().view(grid[0], 8).tolist()
def med(f): v = [f(r) / 1e3 for r in d]; return [round(statistics.median(v), 2), round(max(v), 2)]
print(json.dumps({"loop(warp0)": med(lambda r: r[1] - r[0]), "wait_full": med(lambda r: r[2]), "qk": med(lambda r: r[3]),
                  "sync": med(lambda r: r[4]), "pv": med(lambda r: r[5]), "producer": med(lambda r: r[7]), "tail": med(lambda r: r[6] - r[1])}))
dom.stop(); dom.close()
