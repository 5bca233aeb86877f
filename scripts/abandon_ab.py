"""Config 2 A/B: the training GEMM with and without sub-block yields."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fractions import Fraction
import bench

co = bench.Colocation(0, 8, 1024, decode_sat=Fraction(1, 2),
                      tiers=[Fraction(1, 4), Fraction(1, 2), Fraction(3, 4), Fraction(1)], abandon=True)
solo = co.solo(steps=3)
reqs = int(os.environ.get("REQS", "20"))
rows = []
for rep in range(2):
    for name, k in (("plain", co.gemm_kernel_plain), ("abandon", co.gemm_kernel_abandon)):
        co.gemm_kernel = k
        r = co.run("tpot-first", reqs, 3, solo)
        tm = co.run("temporal", reqs, 3, solo) if (rep == 0 and name == "plain") else None
        row = {"gemm": name, "p99_tpot_ms": round(bench.nearest_rank(r["tpot_ms"], 99), 3),
               "train_tflops": round(r["train_tflops"], 1), "step_ms": round(r["step_ms"], 3)}
        if tm:
            row["temporal_p99_tpot_ms"] = round(bench.nearest_rank(tm["tpot_ms"], 99), 3)
            row["temporal_train_tflops"] = round(tm["train_tflops"], 1)
        rows.append(row)
        print(json.dumps(row), flush=True)
co.gemm_kernel = co.gemm_kernel_plain
print("bit_exact", co.bit_exact_check())
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open("gpurun_out/abandon_ab.json", "w"), indent=1)
co.close()
