"""Decode step on the executor (148 SMs) vs the early-start L2 prefetch depth
per projection (GemvArgs.l2_pf_kb).  One model, one Domain per setting."""
import os, sys, json, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig

m = DecodeModel(DecodeConfig())
tok0 = m.tokens.clone()
torch.cuda.synchronize()
KEYS = {"decode/attn": "attn", "decode/qkv": "qkv", "decode/o": "o", "decode/gate_up": "gu", "decode/down": "down", "decode/lm_head": "lm"}
configs = [x for x in os.environ.get("PF_CONFIGS", "none;all:128;all:256;all:512;all:1024").split(";")]
ref = None
for cfg in configs:
    pf = {k: 0 for k in KEYS.values()}
    for kv in filter(None, cfg.split(",")):
        if kv == "none":
            continue
        k, v = kv.split(":")
        for kk in (pf if k == "all" else [k]):
            pf[kk] = int(v)
    for sid, body, grid, args, _ in m.records:
        if sid in KEYS:
            args.l2_pf_kb = pf[KEYS[sid]]
    m.tokens.copy_(tok0); torch.cuda.synchronize()
    dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=1 << 16)
    t = dom.tenant("decode", _abi.LATENCY_CRITICAL)
    kids = m.register(dom)
    dom.start()
    dom.quota_set(dom.mask(t, 0, dom.num_sms))
    for i in range(2):
        for k in kids: last = dom.launch(t, k)
    dom.wait(t, last); dom.poll(); dom.clear_logs()
    steps = 8
    for i in range(steps):
        for k in kids: last = dom.launch(t, k)
    dom.wait(t, last)
    cs = dom.poll(100000)
    ends = [c.t_end for c in cs]
    n = len(kids)
    per_step = sorted((ends[(i + 1) * n - 1] - ends[i * n - 1]) / 1e6 for i in range(1, steps))
    by = collections.defaultdict(list)
    for i, c in enumerate(cs):
        by[m.records[i % n][0]].append((c.t_end - c.t_first_claim) / 1e3)
    out = m.logits.clone()
    dom.stop(); dom.close()
    same = None if ref is None else bool(torch.equal(out, ref))
    if ref is None: ref = out
    print(json.dumps({"pf": pf, "step_ms_med": per_step[len(per_step) // 2], "step_ms_min": per_step[0],
                      "GBps": m.step_bytes / (per_step[len(per_step) // 2] * 1e-3) / 1e9, "logits_same": same,
                      "span_us": {k: round(sum(v) / len(v), 1) for k, v in by.items()}}), flush=True)
