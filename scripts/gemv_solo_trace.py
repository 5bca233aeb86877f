"""Per-block phase stamps of one decode GEMV as a plain-grid solo launch
(GemvArgs.dbg): block start spread (launch ramp), mainloop (start ->
accumulator final), epilogue, end -- where a solo launch's time goes
beyond its bytes / HBM peak."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import solo_launch
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
m = DecodeModel(DecodeConfig(layers=2))
out = {}
for kname in os.environ.get("KERNELS", "gate_up,down,qkv,o").split(","):
    i = [r[0] for r in m.records].index("decode/" + kname)
    sid, body, grid, args, nbytes = m.records[i]
    G = grid[0] * grid[1] * grid[2]
    d = torch.zeros(G * 8, dtype=torch.int64, device="cuda")
    args.dbg = d.data_ptr()
    for _ in range(3):
        solo_launch(0, sid, body, grid, args)
    torch.cuda.synchronize()
    d.zero_()
    solo_launch(0, sid, body, grid, args)
    torch.cuda.synchronize()
    args.dbg = 0
    x = d.view(G, 8).cpu().numpy().astype("int64") & ((1 << 62) - 1)
    t0 = x[:, 0].min()
    rel = (x - t0) / 1e3
    span = (x[:, 6].max() - t0) / 1e3
    out[kname] = {"blocks": G, "span_us": round(span, 2), "GBps_span": round(nbytes / (span * 1e3), 1),
                  "start_spread_us": [round(float(v), 2) for v in (rel[:, 0].min(), statistics.median(rel[:, 0]), rel[:, 0].max())],
                  "mainloop_us_med": round(float(statistics.median(rel[:, 1] - rel[:, 0])), 2),
                  "epilogue_us_med": round(float(statistics.median(rel[:, 5] - rel[:, 1])), 2),
                  "epi_to_scale_us_med": round(float(statistics.median(rel[:, 4] - rel[:, 1])), 2) if x[:, 4].max() > 0 else None,
                  "epi_mode_us_med": round(float(statistics.median(rel[:, 5] - rel[:, 4])), 2) if x[:, 4].max() > 0 else None,
                  "teardown_us_med": round(float(statistics.median(rel[:, 6] - rel[:, 5])), 2),
                  "accum_final_us": [round(float(v), 2) for v in (rel[:, 1].min(), statistics.median(rel[:, 1]), rel[:, 1].max())],
                  "end_us": [round(float(v), 2) for v in (rel[:, 6].min(), statistics.median(rel[:, 6]), rel[:, 6].max())]}
    own = x[:, 2] > 0  # combiners (split-K owners) stamp the partials-arrived time
    if own.any():
        r = rel[own]
        out[kname]["owners"] = {
            "n": int(own.sum()),
            "wait_partials_us_med": round(float(statistics.median(((x[own, 2] - t0) / 1e3) - r[:, 1])), 2),
            "sum_us_med": round(float(statistics.median(r[:, 3] - (x[own, 2] - t0) / 1e3)), 2),
            "scale_us_med": round(float(statistics.median(r[:, 4] - r[:, 3])), 2),
            "mode_us_med": round(float(statistics.median(r[:, 5] - r[:, 4])), 2),
            "end_us_max": round(float(r[:, 6].max()), 2)}
    print(kname, json.dumps(out[kname]), flush=True)
