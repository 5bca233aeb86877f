"""Which 74 SMs should a half-GPU decode quota get?  Decode step time (and
GEMM time on the complement, co-running) for different SM selections:
contiguous smid ranges vs TPC-interleaved vs strided."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig, TrainGemm

m = DecodeModel(DecodeConfig(layers=int(os.environ.get("LAYERS", "32"))))
tr = TrainGemm()
torch.cuda.synchronize()
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=0)
td = dom.tenant("decode", _abi.LATENCY_CRITICAL)
tt = dom.tenant("train", _abi.BEST_EFFORT)
kids = m.register(dom)
gk = tr.register(dom)
dom.start()
N = dom.num_sms
smids = dom.smids()
slot_of = {sm: i for i, sm in enumerate(smids)}
print("smids by slot", smids, flush=True)
STASH = []


def poll(t):
    STASH.extend(dom.poll(1 << 20))
    mine = [c for c in STASH if c.tenant == t]
    STASH[:] = [c for c in STASH if c.tenant != t]
    return mine


def decode_steps(steps=3):
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


sorted_sm = sorted(smids)
layouts = {
    "slot_order_first74": [smids[i] for i in range(74)],
    "smid_0_73": sorted_sm[:74],
    "smid_74_147": sorted_sm[74:],
    "tpc_even": [s for s in sorted_sm if (s // 2) % 2 == 0][:74],
    "sm_even": [s for s in sorted_sm if s % 2 == 0][:74],
    "smid_mod4_lt2": [s for s in sorted_sm if s % 4 < 2][:74],
    "tpc_block8": [s for s in sorted_sm if (s // 16) % 2 == 0][:74],
}
out = {}
for name, sel in layouts.items():
    sel = set(sel)
    owner = [td if smids[i] in sel else tt for i in range(N)]
    dom.quota_set(owner, [-1] * N)
    solo = decode_steps()
    poll(tt)
    for _ in range(10): lastg = dom.launch(tt, gk)
    co = decode_steps(3)
    dom.wait(tt, lastg)
    g = [(c.t_end - c.t_first_claim) / 1e6 for c in poll(tt)]
    out[name] = {"n": len(sel), "decode_ms": round(solo, 3), "decode_ms_colo": round(co, 3),
                 "gemm_ms_colo": round(statistics.median(g), 3)}
    print(name, out[name], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump({"smids": smids, "layouts": out}, open("gpurun_out/sm_layout.json", "w"), indent=1)
dom.stop(); dom.close()
