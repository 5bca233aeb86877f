"""ResNet-50-shaped training stream (config 4) through the executor on the
full GPU: iteration time, achieved TFLOP/s, slowest GEMMs."""
import os, sys, json, statistics, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import ResNetStream

rs = ResNetStream()
torch.cuda.synchronize()
print("launches/iter", len(rs.records), "TFLOP/iter", rs.flops / 1e12, "padded", rs.padded_flops / 1e12, flush=True)
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=0)
t = dom.tenant("train", _abi.BEST_EFFORT)
kids = rs.register(dom)
dom.start()
dom.quota_set(dom.mask(t, 0, dom.num_sms))
for k in kids: last = dom.launch(t, k)
dom.wait(t, last); dom.poll(1 << 20)
iters = 3
for _ in range(iters):
    for k in kids: last = dom.launch(t, k)
dom.wait(t, last)
cs = dom.poll(1 << 20)
n = len(kids)
it = [(cs[(i + 1) * n - 1].t_end - cs[i * n].t_first_claim) / 1e6 for i in range(iters)]
ms = statistics.median(it)
per = collections.defaultdict(list)
for i, c in enumerate(cs):
    start = c.t_first_claim if i == 0 else max(c.t_first_claim, cs[i - 1].t_end)
    per[rs.records[i % n][0]].append((c.t_end - start) / 1e3)
rows = sorted(((statistics.median(v), k) for k, v in per.items()), reverse=True)
fl = {r[0]: r[4] for r in rs.records}
# per-GEMM lower bound: max(flops / bf16 peak, operand + output bytes / HBM peak)
pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
shape = {f"resnet/{nm}": (M, N, K) for nm, M, N, K in rs.gemms}
def bound_us(k):
    if k not in shape: return 0.0
    M, N, K = shape[k]
    return max(2.0 * M * N * K / (pk["bf16_tflops"] * 1e12), 2.0 * (M * K + N * K + M * N) / (pk["hbm_gbs"] * 1e9)) * 1e6
allrows = sorted(((statistics.median(v) - bound_us(k), statistics.median(v), bound_us(k), k) for k, v in per.items()), reverse=True)
out = {"iter_ms": ms, "tflops": rs.flops / (ms * 1e-3) / 1e12, "images_per_s": rs.batch / (ms * 1e-3),
       "bound_ms": sum(bound_us(k) for k in per) / 1e3,
       "top": [(k, round(us, 1), round(fl[k] / (us * 1e-6) / 1e12, 1)) for us, k in rows[:15]],
       "by_excess_us": [(k, round(us, 1), round(b, 1), rs.plans[[r[0] for r in rs.records if not r[0].endswith("/fold")].index(k)]
                         if k in shape else None) for ex, us, b, k in allrows]}
print(json.dumps(out, indent=0), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/perf_resnet.json", "w"), indent=1)
dom.stop(); dom.close()
