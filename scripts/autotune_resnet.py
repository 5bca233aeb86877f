"""Per-GEMM (tile width, split-K, tiles per block) search for every GEMM of
the ResNet stream: each candidate runs as its GEMM (+ fold) launch pair
on the full-GPU executor (5 timed pairs, median of first-claim -> fold end);
the fastest is written to paper_2603_15042_b200/resnet_plan.json, which
ResNetStream applies (DS_RESNET_TUNED=0 ignores it).  Reduction order is a
function of the chosen record, so solo and coroutine runs stay bit-identical."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["DS_RESNET_TUNED"] = "0"
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain
from paper_2603_15042_b200.tenants import ResNetStream, plan_gemm, WORKERS, _round

rs = ResNetStream()
WS = torch.zeros(96 << 20, device="cuda")  # 384 MB fp32 workspace for the candidates
dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=0)
t = dom.tenant("train", _abi.BEST_EFFORT)
dom.start()
dom.quota_set(dom.mask(t, 0, dom.num_sms))


def time_pair(Mp, Np, Kp, bn, S, T=1):
    ga = _abi.gemm_args(rs.A.data_ptr(), rs.B.data_ptr(), rs.C.data_ptr(), Mp, Np, Kp, bn=bn, splits=S,
                        ws=WS.data_ptr() if S > 1 else 0, tiles=T)
    ks = [dom.kernel("tune/gemm", _abi.BODY_GEMM_BF16, _abi.gemm_grid(Mp, Np, bn, S, T), ga)]
    if S > 1:
        ra, rg = _abi.splitk_reduce(WS.data_ptr(), rs.C.data_ptr(), Mp, Np, Kp, 16, bn, S,
                                    _abi.fold_rows(Mp, Np, bn, WORKERS))
        ks.append(dom.kernel("tune/fold", _abi.BODY_SPLITK_REDUCE, rg, ra))
    for _ in range(2):
        for k in ks: last = dom.launch(t, k)
    dom.wait(t, last); dom.poll(1 << 16)
    ts = []
    for _ in range(5):
        seqs = [dom.launch(t, k) for k in ks]
        dom.wait(t, seqs[-1])
        cs = [c for c in dom.poll(1 << 16) if c.tenant == t]
        ts.append((cs[-1].t_end - cs[0].t_first_claim) / 1e3)
    return statistics.median(ts)


from paper_2603_15042_b200.tenants import plan_tiles
table = {}
for name, M, N, K in rs.gemms:
    Mp, Np, Kp, bn0, S0 = plan_gemm(M, N, K)
    bnT, T0 = plan_tiles(Mp, Np, Kp, bn0, S0, max_tiles=4)
    base = (bnT, S0, T0)  # the heuristic plan as the stream builds it
    cands = {base}
    for bn in (64, 128, 256):
        if Np % bn:
            continue
        tiles = (Mp // 128) * (Np // bn)
        for S in {1, max(2, S0 // 2), S0, 2 * S0, -(-WORKERS // tiles), -(-2 * WORKERS // tiles)}:
            if S > 1 and ((Kp // 64) // S < 8 or _abi.splitk_ws_elems(Mp, Np, bn, S) > WS.numel()):
                continue
            if S == 1 and tiles < WORKERS // 2:
                continue  # far below a wave: not a candidate
            cands.add((bn, S, 1))
            if S == 1 and bn <= 128 and Kp <= 1152:
                for T in (2, 4, 8):
                    if tiles // T >= WORKERS:
                        cands.add((bn, 1, T))
    res = {c: time_pair(Mp, Np, Kp, *c) for c in sorted(cands)}
    best = min(res, key=res.get)
    table[name] = {"bn": best[0], "splits": best[1], "tiles": best[2], "us": round(res[best], 1),
                   "plan": list(base), "plan_us": round(res[base], 1)}
    print(name, table[name], flush=True)
dom.stop(); dom.close()
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2603_15042_b200", "resnet_plan.json")
json.dump(table, open(out, "w"), indent=1)
json.dump(table, open("gpurun_out/resnet_plan.json", "w"), indent=1)
print("gain_us", round(sum(v["plan_us"] - v["us"] for v in table.values()), 1))
