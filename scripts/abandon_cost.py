"""Unflipped throughput of the training GEMM tile with and without the
abandon checks (same domain, back-to-back launches)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fractions import Fraction
import torch
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import TrainGemm
g = TrainGemm(M=16384, N=16384, K=8192, seed=5)
ab = _abi.gemm_args(g.A.data_ptr(), g.B.data_ptr(), g.C.data_ptr(), 16384, 16384, 8192, group_m=32, abandon=True)
torch.cuda.synchronize()
with Domain(0, tiers=[Fraction(1)], block_log_capacity=0, lend_idle_sms=False) as dom:
    t = dom.tenant("t", 1)
    if os.environ.get("MARK", "1") == "1":
        dom.set_abandonable(t)
    kp = g.register(dom)
    ka = dom.kernel("ab", _abi.BODY_GEMM_BF16, g.grid, ab)
    dom.start()
    dom.quota_set([t] * dom.num_sms)
    for name, k in (("plain", kp), ("abandon", ka), ("plain", kp), ("abandon", ka)):
        dom.poll(1 << 16)
        for _ in range(3):
            last = dom.launch(t, k)
        dom.wait(t, last)
        cs = [c for c in dom.poll(1 << 16) if c.tenant == t]
        ms = statistics.median([(c.t_end - c.t_first_claim) / 1e6 for c in cs[-3:]])
        print(name, round(ms, 3), "ms", round(2 * 16384 * 16384 * 8192 / ms / 1e9, 1), "TF/s", flush=True)
