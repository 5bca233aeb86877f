"""Decode step time and GEMM time as a function of the SM quota, solo and
co-located (decode on the first X SMs, GEMM on the rest, both running).
Tells how many SMs the HBM-bound decode tenant needs."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig, TrainGemm

layers = int(os.environ.get("LAYERS", "32"))
m = DecodeModel(DecodeConfig(layers=layers))
tr = TrainGemm()
torch.cuda.synchronize()
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=0)
td = dom.tenant("decode", _abi.LATENCY_CRITICAL)
tt = dom.tenant("train", _abi.BEST_EFFORT)
kids = m.register(dom)
gk = tr.register(dom)
dom.start()
N = dom.num_sms


STASH = []


def poll(t):
    STASH.extend(dom.poll(1 << 20))
    mine = [c for c in STASH if c.tenant == t]
    STASH[:] = [c for c in STASH if c.tenant != t]
    return mine


def decode_steps(steps=4):
    for k in kids: last = dom.launch(td, k)
    dom.wait(td, last)
    poll(td)
    for _ in range(steps):
        for k in kids: last = dom.launch(td, k)
    dom.wait(td, last)
    cs = poll(td)
    n = len(kids)
    ends = [cs[(i + 1) * n - 1].t_end for i in range(steps)]
    return statistics.median([(ends[i] - ends[i - 1]) / 1e6 for i in range(1, steps)])


def gemm_rate(iters=4):
    poll(tt)
    for _ in range(iters): last = dom.launch(tt, gk)
    dom.wait(tt, last)
    cs = poll(tt)
    return statistics.median([(c.t_end - c.t_first_claim) / 1e6 for c in cs])


out = []
for x in [148, 128, 111, 96, 74, 56, 37]:
    owner = [td] * x + [tt] * (N - x)
    dom.quota_set(owner, [-1] * N)
    solo_dec = decode_steps()
    row = {"decode_sms": x, "decode_step_ms": round(solo_dec, 3), "decode_GBps": round(m.step_bytes / solo_dec / 1e6, 1)}
    if x < N:
        row["gemm_ms_rest_solo"] = round(gemm_rate(), 3)
        # co-located: keep GEMMs queued while decode steps run
        poll(tt)
        for _ in range(12): lastg = dom.launch(tt, gk)
        co_dec = decode_steps(3)
        dom.wait(tt, lastg)
        cs = poll(tt)
        row["decode_step_ms_colo"] = round(co_dec, 3)
        g = [(c.t_end - c.t_first_claim) / 1e6 for c in cs]
        row["gemm_ms_colo_median"] = round(statistics.median(g), 3)
    print(json.dumps(row), flush=True)
    out.append(row)
dom.quota_set([tt] * N, [-1] * N)
row = {"gemm_ms_full": round(gemm_rate(), 3)}
print(json.dumps(row), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out + [row], open("gpurun_out/quota_curve.json", "w"), indent=1)
dom.stop(); dom.close()
