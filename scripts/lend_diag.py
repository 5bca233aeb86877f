"""Where does idle-SM lending cost decode time?  A short TPOT-First
co-located run with the block log on: per decode step, the SMs the decode
launches ran on, the training blocks that ran on those SMs inside the step,
and the control-word changes (ctl log) inside the step."""
import os, sys, json, statistics, collections
os.environ.setdefault("DS_BENCH_BLOG", str(1 << 23))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from fractions import Fraction
co = bench.Colocation(0, 8, 1024, layers=32, decode_sat=Fraction(1, 2), slo_x=8.0,
                      tiers=[Fraction(1, 4), Fraction(1, 2), Fraction(3, 4), Fraction(1)])
solo = co.solo(steps=3)
dom = co.dom
dom.block_log()  # drain
res = co.run("tpot-first", int(os.environ.get("REQ", "12")), 2, solo)
blog = dom.block_log()
td, tt = co.t_dec, co.t_trn
dec = [b for b in blog if b.tenant == td]
trn = [b for b in blog if b.tenant == tt]
print("blocks", len(dec), len(trn), "tpot p50", statistics.median(res["tpot_ms"]))
# decode steps = runs of 163 launches; group decode blocks by seq
by_seq = collections.defaultdict(list)
for b in dec:
    by_seq[b.seq].append(b)
seqs = sorted(by_seq)
nk = len(co.dec_kernels_half)
steps = [seqs[i:i + nk] for i in range(0, len(seqs) - nk + 1, nk)]
rows = []
for st in steps[-40:]:
    bs = [b for s in st for b in by_seq[s]]
    t0, t1 = min(b.t_start for b in bs), max(b.t_end for b in bs)
    sms = set(b.smid for b in bs)
    intr = [b for b in trn if b.smid in sms and b.t_start < t1 and b.t_end > t0]
    intr_us = sum(min(b.t_end, t1) - max(b.t_start, t0) for b in intr) / 1e3
    rows.append({"step_ms": (t1 - t0) / 1e6, "dec_sms": len(sms), "trn_blocks_on_dec_sms": len(intr),
                 "trn_us_on_dec_sms": round(intr_us, 1),
                 "trn_started_inside": sum(1 for b in intr if b.t_start > t0)})
for r in rows[-10:]:
    print(r)
out = {k: statistics.median(r[k] for r in rows) for k in rows[0]}
print("median", out)
json.dump({"rows": rows, "median": out}, open("gpurun_out/lend_diag.json", "w"), indent=1)
co.close()
