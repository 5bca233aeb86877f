"""Per-block timeline of decode kernels under the executor (full GPU)."""
import os, sys, json, statistics, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
m = DecodeModel(DecodeConfig(layers=2))
torch.cuda.synchronize()
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=1 << 22)
t = dom.tenant("decode", _abi.LATENCY_CRITICAL)
kids = m.register(dom)
dom.start()
dom.quota_set(dom.mask(t, 0, dom.num_sms))
names = [r[0] for r in m.records]
for name in ("decode/qkv", "decode/o", "decode/gate_up", "decode/down", "decode/attn", "decode/lm_head"):
    i = names.index(name)
    k = kids[i]
    rep = 12
    for _ in range(4): last = dom.launch(t, k)
    dom.wait(t, last); dom.poll(1 << 16); dom.clear_logs()
    s0 = last + 1
    for _ in range(rep): last = dom.launch(t, k)
    dom.wait(t, last)
    cs = dom.poll(1 << 16)
    bl = [b for b in dom.block_log() if b.tenant == t]
    durs = [(c.t_end - c.t_first_claim) / 1e3 for c in cs]
    span = (cs[-1].t_end - cs[0].t_first_claim) / 1e3 / rep
    one = [b for b in bl if b.seq == s0 + rep // 2]
    k0 = min(b.t_start for b in one)
    starts = sorted((b.t_start - k0) / 1e3 for b in one)
    bd = sorted((b.t_end - b.t_start) / 1e3 for b in one)
    bytes_ = m.records[i][4]
    print(json.dumps({"kernel": name, "blocks": len(one), "launch_us_med": statistics.median(durs),
                      "steady_us_per_launch": span, "GBps_steady": bytes_ / (span * 1e3),
                      "start_offsets_us(p0,p50,p90,max)": [starts[0], starts[len(starts)//2], starts[int(len(starts)*.9)], starts[-1]],
                      "block_us(p10,p50,p90,max)": [bd[len(bd)//10], bd[len(bd)//2], bd[int(len(bd)*.9)], bd[-1]]}), flush=True)
dom.stop(); dom.close()
