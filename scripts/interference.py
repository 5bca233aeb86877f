"""Decode step at 74 SMs beside a training GEMM on the other 74 SMs, per GEMM
tile configuration: how much of the co-located slowdown follows the GEMM's
memory traffic.  Raw domain, no policy: decode owns SMs [0, 74), training
[74, 148)."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig, TrainGemm

m = DecodeModel(DecodeConfig(layers=int(os.environ.get("LAYERS", "32"))))
tg = TrainGemm()
variants = {"none": None,
            "bn256_gm32": _abi.gemm_args(tg.A.data_ptr(), tg.B.data_ptr(), tg.C.data_ptr(), 8192, 8192, 8192, group_m=32),
            "bn256_gm8": _abi.gemm_args(tg.A.data_ptr(), tg.B.data_ptr(), tg.C.data_ptr(), 8192, 8192, 8192, group_m=8),
            "bn256_gm64": _abi.gemm_args(tg.A.data_ptr(), tg.B.data_ptr(), tg.C.data_ptr(), 8192, 8192, 8192, group_m=64),
            "bn128_gm32": _abi.gemm_args(tg.A.data_ptr(), tg.B.data_ptr(), tg.C.data_ptr(), 8192, 8192, 8192, group_m=32,
                                         bn=128)}
torch.cuda.synchronize()
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=0, lend_idle_sms=False)
td = dom.tenant("decode", 0)
tt = dom.tenant("train", 1)
kids = m.register(dom)
gk = {}
for name, a in variants.items():
    if a is None:
        continue
    bn = a.bn or 256
    gk[name] = dom.kernel("train/" + name, _abi.BODY_GEMM_BF16, _abi.gemm_grid(8192, 8192, bn), a)
dom.start()
n = dom.num_sms
smids = dom.smids()
order = sorted(range(n), key=lambda i: smids[i])
low = set(order[: n // 2])  # the engine's pick_slots: lowest smids (whole TPCs) first
dn = int(os.environ.get("DEC_SMS", n // 2))  # decode's SM count (slot order)
layouts = {f"slot_order_{dn}": [td if i < dn else tt for i in range(n)]}
_unused = {
           "low_smids": [td if i in low else tt for i in range(n)],
           "even_smids": [td if smids[i] % 4 < 2 else tt for i in range(n)]}
if os.environ.get("LAYOUTS"):
    layouts = {k: v for k, v in layouts.items() if k in os.environ["LAYOUTS"].split(",")}
only = os.environ.get("VARIANTS", "")
if only:
    variants = {k: v for k, v in variants.items() if k in only.split(",")}
res = {}
for (lname, owner), name in [(lo, v) for lo in layouts.items() for v in variants]:
    dom.quota_set(owner)
    tseqs = []
    if name != "none":
        tseqs = [dom.launch(tt, gk[name]) for _ in range(int(os.environ.get("GEMMS", "70")))]
    for k in kids:
        last = dom.launch(td, k)
    dom.wait(td, last)
    dom.poll(1 << 20)
    steps = []
    for _ in range(int(os.environ.get("STEPS", "6"))):
        for k in kids:
            last = dom.launch(td, k)
        dom.wait(td, last)
        cs = [c for c in dom.poll(1 << 20)]
        dc = [c for c in cs if c.tenant == td]
        steps.append((dc[-1].t_end - dc[0].t_first_claim) / 1e6)
    tf = None
    if tseqs:
        dom.wait(tt, tseqs[-1], 120000)
        tc = [c for c in dom.poll(1 << 20) if c.tenant == tt]
    res[lname + "/" + name] = {"decode_step_ms": round(statistics.median(steps), 3),
                               "first_last": [round(steps[0], 3), round(steps[-1], 3)]}
    print(lname + "/" + name, res[lname + "/" + name], flush=True)
print("smids of the first 8 slots", smids[:8])
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/interference.json", "w"), indent=1)
dom.stop()
dom.close()
