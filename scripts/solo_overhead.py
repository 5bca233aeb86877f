"""Fixed cost of a plain-grid solo launch: the spin test body (no TMEM, no
smem ring) at 128 CTAs with a 1-us spin vs the decode o projection; run
under ncu for gpu__time_duration, and with ds_solo_trace for the CTA span."""
import os, sys, json, ctypes, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200._abi import lib, check
from paper_2603_15042_b200.runtime import solo_launch
out = torch.zeros(128 * 4, dtype=torch.int64, device="cuda")
sa = _abi.SpinArgs()
for f, _ in sa._fields_:
    pass
sa.ns = 1000
if hasattr(sa, "out"):
    sa.out = out.data_ptr()
buf = torch.zeros(128 * 4, dtype=torch.int64, device="cuda")
for _ in range(3): solo_launch(0, "spin", _abi.BODY_SPIN, (128, 1, 1), sa)
torch.cuda.synchronize()
if not os.environ.get("NCU"):
    check(lib().ds_solo_trace(0, ctypes.c_void_p(buf.data_ptr())))
solo_launch(0, "spin", _abi.BODY_SPIN, (128, 1, 1), sa)
torch.cuda.synchronize()
check(lib().ds_solo_trace(0, None))
if not os.environ.get("NCU"):
    x = buf.view(128, 4).cpu().numpy().astype("int64")
    r = (x - x[:, 0].min()) / 1e3
    print("spin cta_span_us", round(float(r[:, 3].max()), 2), "body med", round(float(statistics.median(r[:, 2] - r[:, 1])), 2))
