"""Decode step on a half-GPU quota: back-to-back launches vs one step at a
time vs records dispatched by the policy engine (no training tenant)."""
import os, sys, json, statistics, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain, Engine
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig

m = DecodeModel(DecodeConfig(layers=int(os.environ.get("LAYERS", "32"))))
torch.cuda.synchronize()
tiers = [Fraction(1, 4), Fraction(1, 2), Fraction(3, 4), Fraction(1)]
dom = Domain(0, tiers=tiers, block_log_capacity=0, lend_idle_sms=True)
td = dom.tenant("decode", _abi.LATENCY_CRITICAL)
kids = m.register(dom)
dom.start()
N = dom.num_sms
res = {}
dom.quota_set([td] * 74 + [-1] * (N - 74), [-1] * N)
# (a) back-to-back
for k in kids: last = dom.launch(td, k)
dom.wait(td, last); dom.poll(1 << 20)
for _ in range(4):
    for k in kids: last = dom.launch(td, k)
dom.wait(td, last)
cs = dom.poll(1 << 20)
n = len(kids)
res["b2b_step_ms"] = statistics.median([(cs[(i + 1) * n - 1].t_end - cs[i * n].t_first_claim) / 1e6 for i in range(4)])
res["b2b_period_ms"] = statistics.median([(cs[(i + 1) * n - 1].t_end - cs[i * n - 1].t_end) / 1e6 for i in range(1, 4)])
# (b) one step at a time
st = []
for _ in range(4):
    for k in kids: last = dom.launch(td, k)
    dom.wait(td, last)
    cs = dom.poll(1 << 20)
    st.append((cs[-1].t_end - cs[0].t_first_claim) / 1e6)
res["single_step_ms"] = statistics.median(st)
# per-kernel first-claim lag behind previous completion (loader / early-start)
lag = [(cs[i].t_first_claim - cs[i - 1].t_end) / 1e3 for i in range(1, n)]
res["kernel_gap_us_mean"] = statistics.mean(lag)
res["kernel_gap_us_max"] = max(lag)
dom.quota_set([-1] * N, [-1] * N)
# (c) engine
eng = Engine(dom, policy="tpot-first", lend_tenant=-1)
jd = eng.add_job(td, _abi.LATENCY_CRITICAL)
eng.start()
recs = []
for tok in range(6):
    recs.append(eng.submit(jd, kids, "decode/step", _abi.DECODE, grid_size=len(kids), request=0, decode_index=tok,
                           tpot_ns=10**9, ttft_ns=10**9, base_hint_ns=9_000_000, saturation=Fraction(1, 2)))
eng.wait(recs[-1])
infos = [eng.record(r) for r in recs]
res["engine_step_ms"] = statistics.median([(i.t_end - i.t_first_claim) / 1e6 for i in infos[1:]])
res["engine_gap_us"] = statistics.median([(infos[i + 1].t_first_claim - infos[i].t_end) / 1e3 for i in range(5)])
res["engine_pctx"] = [i.pctx for i in infos]
eng.stop(); eng.close()
print(json.dumps(res), flush=True)
dom.stop(); dom.close()
