"""Solo and coroutine throughput of the tcgen05 GEMM tenant (8192^3 bf16)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain, solo_launch
from paper_2603_15042_b200._abi import lib, check
import ctypes
M = N = K = int(os.environ.get("SZ", "8192"))
A = (torch.rand(M, K, device="cuda") * 2 - 1).to(torch.bfloat16)
B = (torch.rand(N, K, device="cuda") * 2 - 1).to(torch.bfloat16)
C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
BN = int(os.environ.get("BN", "256"))
BK = int(os.environ.get("BK", "64"))
GM = int(os.environ.get("GM", "16"))
args = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, group_m=GM, bn=BN, bk=BK)
grid = _abi.gemm_grid(M, N, BN)
flop = 2.0 * M * N * K
desc = __import__("paper_2603_15042_b200.runtime", fromlist=["make_desc"]).make_desc("gemm", _abi.BODY_GEMM_BF16, grid, args)
for i in range(3):
    check(lib().ds_solo_launch(0, ctypes.byref(desc), None))
torch.cuda.synchronize()
ts = []
for i in range(5):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); check(lib().ds_solo_launch(0, ctypes.byref(desc), None)); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ref = (A[:256].float() @ B.float().t()[:, :512])
err = float(((C[:256, :512].float() - ref).abs() / (ref.abs() + 1)).max())
cub = []
for i in range(5):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); torch.matmul(A, B.t()); e1.record(); torch.cuda.synchronize(); cub.append(e0.elapsed_time(e1))
print(json.dumps({"solo_ms": ts, "solo_tflops": flop / (min(ts) * 1e-3) / 1e12, "max_rel_err": err,
                  "cublas_ms": min(cub), "cublas_tflops": flop / (min(cub) * 1e-3) / 1e12}))
with Domain(0, block_log_capacity=0) as dom:
    dom.start()
    t = dom.tenant("train", 1)
    dom.quota_set(dom.mask(t, 0, dom.num_sms))
    kid = dom.kernel("gemm", _abi.BODY_GEMM_BF16, grid, args)
    for i in range(3):
        s = dom.launch(t, kid)
    dom.wait(t, s)
    dom.poll()
    n = int(os.environ.get("ITERS", "10"))
    for i in range(n):
        s = dom.launch(t, kid)
    dom.wait(t, s)
    cs = dom.poll()
    t0 = min(c.t_first_claim for c in cs); t1 = max(c.t_end for c in cs)
    per = [(c.t_end - c.t_first_claim) / 1e6 for c in cs]
    import statistics as _st
    print(json.dumps({"sustained_median_ms": _st.median(per[n // 2:]), "coroutine_ms_per_gemm": (t1 - t0) / 1e6 / n, "coroutine_tflops": flop * n / ((t1 - t0) * 1e-9) / 1e12,
                      "per_launch_ms": per[:4], "sms_used": [c.sms_used for c in cs[:3]]}))
