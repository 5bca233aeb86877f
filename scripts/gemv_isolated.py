"""One decode GEMV record launched back to back (nothing else resident) at a
given SM count: per-block duration and per-lane streaming rate, next to the
same record inside a decode step (critpath/block_stats)."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
nsm = int(os.environ.get("NSM", "74"))
m = DecodeModel(DecodeConfig(layers=2))
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=1 << 20)
t = dom.tenant("d", 0)
kids = m.register(dom)
kpair = m.register_variant(dom, kids, "gu_pair")
names = [r[0] for r in m.records]
dom.start()
dom.quota_set(dom.mask(t, 0, nsm))
for label, ids in (("gate_up", kids), ("gate_up_pair", kpair), ("down", kids), ("qkv", kids), ("o", kids), ("attn", kids)):
    base = label.replace("_pair", "")
    i = names.index("decode/" + base)
    k = ids[i]
    nbytes = m.records[i][4]
    for _ in range(3): last = dom.launch(t, k)
    dom.wait(t, last); dom.poll(1 << 16); dom.clear_logs()
    s0 = last + 1
    for _ in range(10): last = dom.launch(t, k)
    dom.wait(t, last)
    cs = dom.poll(1 << 16)
    bl = [b for b in dom.block_log() if b.seq >= s0]
    per_launch = (cs[-1].t_end - cs[0].t_first_claim) / 1e3 / 10
    durs = [(b.t_end - b.t_start) / 1e3 for b in bl]
    nb = len(bl) // 10
    print(json.dumps({"nsm": nsm, "kernel": label, "blocks": nb, "us_per_launch": round(per_launch, 1),
                      "GBps": round(nbytes / per_launch / 1e3, 1), "block_us_med": round(statistics.median(durs), 1),
                      "lane_GBps": round(nbytes / nb / statistics.median(durs) / 1e3, 1)}), flush=True)
dom.stop(); dom.close()
