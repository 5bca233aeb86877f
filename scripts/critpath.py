"""Critical path of a decode step on the executor: per launch, the increment
t_end[k] - t_end[k-1] (the time the step spends on launch k once launch k-1
is complete), averaged per kernel, with the bytes each increment streams."""
import os, sys, json, statistics, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import DecodeModel, DecodeConfig
nsm = int(os.environ.get("NSM", "148"))
m = DecodeModel(DecodeConfig(layers=int(os.environ.get("LAYERS", "32"))), split_override=os.environ.get("SPLITS", ""),
                bm_override=os.environ.get("BMS", ""))
print("S", m.S, "BM", m.BM, flush=True)
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=1 << 22)
t = dom.tenant("decode", 0)
kids = m.register(dom)
if os.environ.get("VARIANTS"):  # e.g. "gu_pair,lm_multi": the decode tier's bit-identical variants
    kids = m.register_variant(dom, kids, os.environ["VARIANTS"])
dom.start()
dom.quota_set(dom.mask(t, 0, nsm))
for _ in range(3):
    for k in kids: last = dom.launch(t, k)
dom.wait(t, last); dom.poll(1 << 16); dom.clear_logs()
s0 = last + 1
for k in kids: last = dom.launch(t, k)
dom.wait(t, last)
cs = dom.poll(1 << 16)
bl = dom.block_log()
byk = collections.defaultdict(list)
for b in bl: byk[b.seq].append(b)
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for i in range(1, len(kids)):
    name = m.records[i][0]
    prev_end = cs[i - 1].t_end
    blocks = byk[s0 + i]
    a = agg[name]
    a["incr"].append((cs[i].t_end - prev_end) / 1e3)
    a["first_claim_before_dep"].append((prev_end - min(b.t_start for b in blocks)) / 1e3)
    a["blocks_started_after_dep"].append(sum(b.t_start > prev_end for b in blocks))
    a["last_start_after_dep"].append((max(b.t_start for b in blocks) - prev_end) / 1e3)
    a["tail_last_block_us"].append((cs[i].t_end - max(b.t_start for b in blocks)) / 1e3)
    durs = sorted((b.t_end - b.t_start) / 1e3 for b in blocks)
    a["block_med_us"].append(durs[len(durs) // 2]); a["block_max_us"].append(durs[-1])
    a["nblocks"].append(len(blocks))
tot = (cs[-1].t_end - cs[0].t_end) / 1e3
print("step_us (embed end -> argmax end)", round(tot, 1))
for name, a in agg.items():
    b = next(r[4] for r in m.records if r[0] == name)
    inc = statistics.mean(a["incr"])
    print(json.dumps({"k": name, "n": len(a["incr"]), "incr_us": round(inc, 1), "GBps_incr": round(b / inc / 1e3, 1),
                      **{k: round(statistics.mean(v), 1) for k, v in a.items() if k != "incr"}}), flush=True)
dom.stop(); dom.close()
