import sys, os
sys.path.insert(0, "/root/repo")
from fractions import Fraction
import numpy as np, torch
from paper_2603_15042_b200 import _abi, migration as mg
from paper_2603_15042_b200.runtime import Domain
M, N, K = 4096, 4096, 8192
g = torch.Generator(device="cuda").manual_seed(7)
A = (torch.rand(M, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
B = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
C = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
a = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, group_m=16, abandon=True)
grid = _abi.gemm_grid(M, N)
torch.cuda.synchronize()
with Domain(0, tiers=[Fraction(1)], block_log_capacity=1 << 18) as dom:
    t = dom.tenant("train", 1)
    dom.set_abandonable(t)
    kid = dom.kernel("g", _abi.BODY_GEMM_BF16, grid, a)
    dom.start()
    period = int(os.environ.get("P", "50"))
    r = mg.run(dom, t, kid, period)
    blog = [b for b in dom.block_log() if b.tenant == t]
    ctl = sorted(x.t for x in dom.ctl_log() if x.source == 2)
ab = [b for b in blog if b.flags == 1]
ok = [b for b in blog if b.flags == 0]
print("tiles", len(ok), "abandoned", len(ab), "flips", len(ctl))
print("complete tile us p50", np.median([(b.t_end - b.t_start) / 1e3 for b in ok]))
ctl = np.array(ctl)
d = []
for b in ab:
    i = np.searchsorted(ctl, b.t_end) - 1
    if i >= 0: d.append((b.t_end - ctl[i]) / 1e3)
d = np.array(d)
print("abandon end - last flip (us): p10 %.1f p50 %.1f p90 %.1f" % tuple(np.percentile(d, [10, 50, 90])))
print("abandoned attempt duration p50 us", np.median([(b.t_end - b.t_start) / 1e3 for b in ab]))
y = np.array(r["yield_us"]) / 1e3
print("yield p10 %.1f p50 %.1f p90 %.1f n %d" % (*np.percentile(y, [10, 50, 90]), len(y)))
