"""Config 2 with lane split: decode owns every SM's lane 0, training runs on
every SM's lane 1 (ds_set_lane_split), vs the default SM-set split (decode
binds the 1/2 tier).  Prints P99 TPOT, training TF/s and the mean step."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fractions import Fraction
import bench

co = bench.Colocation(0, 8, 1024, decode_sat=Fraction(1, 2),
                      tiers=[Fraction(1, 4), Fraction(1, 2), Fraction(3, 4), Fraction(1)])
solo = co.solo(steps=3)
print("solo", solo["decode_step_ms"], solo["gemm_ms"], flush=True)
reqs = int(os.environ.get("REQS", "12"))
CFGS = [("sets_sat1/2", Fraction(1, 2), 0), ("lanes_sat1_mode1", Fraction(1), 1),
        ("lanes_sat1_mode2", Fraction(1), 2), ("half_lanes_sat1_mode3", Fraction(1), 3),
        ("half_lanes_sat1_mode4", Fraction(1), 4)]
out = []
for name, sat, mode in CFGS:
    co.decode_sat = sat
    co.dom.set_lane_split(mode)
    r = co.run("tpot-first", reqs, 3, solo)
    row = {"cfg": name, "decode_saturation": str(sat), "lane_split": mode,
           "p99_tpot_ms": round(bench.nearest_rank(r["tpot_ms"], 99), 3),
           "train_tflops": round(r["train_tflops"], 1), "step_ms": round(r["step_ms"], 3)}
    out.append(row)
    print(json.dumps(row), flush=True)
co.dom.set_lane_split(0)
exact = co.bit_exact_check()
print("bit_exact", exact)
os.makedirs("gpurun_out", exist_ok=True)
json.dump({"solo": {"decode_step_ms": solo["decode_step_ms"], "gemm_ms": solo["gemm_ms"]}, "requests": reqs,
           "rows": out, "bit_exact_vs_solo": exact}, open("gpurun_out/lane_split.json", "w"), indent=1)
co.close()
