"""Decode step time vs per-projection K-split at 74 and 148 SMs (one
projection varied at a time around the current plan)."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig

layers = int(os.environ.get("LAYERS", "8"))
base = os.environ.get("BASE", "qkv:3,o:3,gu:2,down:5,lm:1")
cands = {"qkv": [1, 2, 3, 4], "o": [1, 2, 3, 4], "gu": [1, 2, 3], "down": [2, 3, 4, 5, 7], "lm": [1, 2]}
if os.environ.get("CANDS"):  # e.g. '{"o": [6, 8], "qkv": [6]}'
    cands = json.loads(os.environ["CANDS"])
only = os.environ.get("ONLY", "")
if only:
    cands = {k: v for k, v in cands.items() if k in only.split(",")}


def step_times(split):
    m = DecodeModel(DecodeConfig(layers=layers), split_override=split, bm_override=os.environ.get("BMS", ""))
    torch.cuda.synchronize()
    dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=0)
    t = dom.tenant("d", 0)
    kids = m.register(dom)
    dom.start()
    out = {}
    for nsm in (74, 148):
        dom.quota_set(dom.mask(t, 0, nsm))
        for k in kids: last = dom.launch(t, k)
        dom.wait(t, last); dom.poll(1 << 20)
        for _ in range(4):
            for k in kids: last = dom.launch(t, k)
        dom.wait(t, last)
        cs = dom.poll(1 << 20)
        n = len(kids)
        ends = [cs[(i + 1) * n - 1].t_end for i in range(4)]
        out[nsm] = statistics.median([(ends[i] - ends[i - 1]) / 1e3 for i in range(1, 4)])
    dom.stop(); dom.close()
    del m
    torch.cuda.empty_cache()
    return out


res = {}
r0 = step_times(base)
print("base", base, r0, flush=True)
res[base] = r0
for k, vals in cands.items():
    for v in vals:
        kv = dict(x.split(":") for x in base.split(","))
        if int(kv[k]) == v:
            continue
        kv[k] = str(v)
        sp = ",".join(f"{a}:{b}" for a, b in kv.items())
        r = step_times(sp)
        res[sp] = r
        print(k, v, r, flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump({k: v for k, v in res.items()}, open("gpurun_out/split_sweep.json", "w"), indent=1)
