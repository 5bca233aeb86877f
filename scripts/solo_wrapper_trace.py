"""Where a plain-grid solo launch of a decode kernel spends its time: per-CTA
stamps of the solo wrapper (ds_solo_trace: entry, TMEM allocated, body
returned, exit) next to the events-timed launch."""
import os, sys, json, statistics, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200._abi import lib, check
from paper_2603_15042_b200.runtime import solo_launch
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
m = DecodeModel(DecodeConfig(layers=2))
names = [r[0] for r in m.records]
for kname in os.environ.get("KERNELS", "gate_up,o,attn").split(","):
    sid, body, grid, args, nbytes = m.records[names.index("decode/" + kname)]
    G = grid[0] * grid[1] * grid[2]
    buf = torch.zeros(G * 4, dtype=torch.int64, device="cuda")
    for _ in range(3): solo_launch(0, sid, body, grid, args)
    torch.cuda.synchronize()
    check(lib().ds_solo_trace(0, ctypes.c_void_p(buf.data_ptr())))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); solo_launch(0, sid, body, grid, args); e1.record()
    torch.cuda.synchronize()
    check(lib().ds_solo_trace(0, None))
    x = buf.view(G, 4).cpu().numpy().astype("int64")
    t0 = x[:, 0].min()
    r = (x - t0) / 1e3
    med = lambda v: round(float(statistics.median(v)), 2)
    print(kname, json.dumps({"events_us": round(e0.elapsed_time(e1) * 1e3, 2), "cta_span_us": round(float(r[:, 3].max()), 2),
                             "entry_spread_us": [round(float(r[:, 0].min()), 2), med(r[:, 0]), round(float(r[:, 0].max()), 2)],
                             "tmem_alloc_us_med": med(r[:, 1] - r[:, 0]), "tmem_alloc_us_max": round(float((r[:, 1] - r[:, 0]).max()), 2),
                             "body_us_med": med(r[:, 2] - r[:, 1]), "exit_us_med": med(r[:, 3] - r[:, 2]),
                             "exit_us_max": round(float((r[:, 3] - r[:, 2]).max()), 2)}), flush=True)
