"""BASELINE config 3: SM-quota migration sweep.

One tenant runs a stream of logical blocks of fixed length (spin body: B us
per block) or bf16 GEMM tiles; the device flips the SM quota between two
control words (100% <-> 25% of the SMs) every P (50 us .. 5 ms) using the
executor's device-timer program (no host round trip).  From the device logs:
  * install latency: control-word install times are the flip instants;
  * yield latency per revoked SM: first switch-away after a flip - flip time
    (an SM leaves only at a logical-block boundary, so <= one block);
  * grant latency: first block of the tenant on a regained SM - flip time;
  * lost throughput: 1 - achieved blocks/s / (solo blocks/s x time-weighted SM fraction).
Also host -> device control latency (mailbox write -> device install).
"""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from fractions import Fraction
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain

def pct(v, q):
    v = sorted(v)
    return v[min(len(v) - 1, int(q * len(v)))] if v else None

def run(dom, t, block_us, period_us, nblocks):
    n = dom.num_sms
    full = dom.mask(t, 0, n)
    quarter = dom.mask(t, 0, n // 4)
    out = torch.from_numpy(np.zeros(3 * nblocks, np.int64)).cuda()
    kid = dom.kernel(f"spin/{block_us}us", _abi.BODY_SPIN, (nblocks, 1, 1), _abi.SpinArgs(out.data_ptr(), int(block_us * 1000)))
    dom.quota_set(full)
    dom.clear_logs()
    if period_us:
        dom.quota_periodic(int(period_us * 1000), full, quarter)  # first flip installs the 25% word
    s = dom.launch(t, kid)
    dom.wait(t, s, 120000)
    dom.quota_periodic(0, full, full)
    c = [x for x in dom.poll(1 << 16) if x.tenant == t][-1]
    ctl = [r for r in dom.ctl_log() if r.source == 2]
    sw = dom.switch_log()
    span = (c.t_end - c.t_first_claim) / 1e9
    smids = dom.smids()
    revocable = set(smids[n // 4:])
    yields, drains, grants = [], [], []
    flips = [r.t for r in ctl if c.t_first_claim <= r.t <= c.t_end]
    if sw:
        arr = np.array([(x.t, x.smid, x.from_tenant, x.to_tenant) for x in sw], dtype=np.int64)
        arr = arr[np.argsort(arr[:, 0], kind="stable")]
        rev = np.isin(arr[:, 1], np.array(sorted(revocable)))
        away = arr[rev & (arr[:, 2] == t)]
        back = arr[rev & (arr[:, 3] == t)]
        for k, ft in enumerate(flips):
            nxt = flips[k + 1] if k + 1 < len(flips) else c.t_end
            src = away if k % 2 == 0 else back
            lo, hi = np.searchsorted(src[:, 0], [ft, nxt])
            seg = src[lo:hi]
            if not len(seg):
                continue
            # per SM: sorted event times after the flip (two worker lanes)
            order = np.lexsort((seg[:, 0], seg[:, 1]))
            seg = seg[order]
            sms, first_idx, counts = np.unique(seg[:, 1], return_index=True, return_counts=True)
            d0 = seg[first_idx, 0] - ft
            if k % 2 == 0:
                yields += d0.tolist()
                two = counts > 1
                drains += (seg[first_idx[two] + 1, 0] - ft).tolist()
            else:
                grants += d0.tolist()
    # time-weighted SM fraction over the kernel span (full until the first flip)
    edges = [c.t_first_claim] + flips + [c.t_end]
    wfrac = 0.0
    for k in range(len(edges) - 1):
        f = 1.0 if k == 0 else (0.25 if (k - 1) % 2 == 0 else 1.0)
        wfrac += f * (edges[k + 1] - edges[k])
    sm_fraction = wfrac / (c.t_end - c.t_first_claim)
    return {"blocks_per_s": nblocks / span, "span_s": span, "flips": len(flips), "yield_us": yields,
            "sm_fraction": sm_fraction,
            "drain_us": drains, "grant_us": grants}

def main():
    torch.cuda.init()
    dom = Domain(0, tiers=[Fraction(1)], block_log_capacity=0, lend_idle_sms=False)
    dom.start()
    t = dom.tenant("train", _abi.BEST_EFFORT)
    res = {"config": "spin blocks on 1 B200; quota flips 100% <-> 25% of SMs by the device timer", "sweep": []}
    for block_us in (5, 20, 50):
        nblk = int(2 * 148 * 2 * 60000 / block_us / 8)  # ~60 ms of work at full quota
        solo = run(dom, t, block_us, 0, nblk)
        for period_us in (50, 100, 200, 500, 1000, 2000, 5000):
            r = run(dom, t, block_us, period_us, nblk)
            frac = r["sm_fraction"]  # time-weighted SM fraction from the device flip times
            lost = 1.0 - r["blocks_per_s"] / (solo["blocks_per_s"] * frac)
            row = {"block_us": block_us, "period_us": period_us, "flips": r["flips"],
                   "yield_us_p50": round(pct(r["yield_us"], .5) / 1e3, 2) if r["yield_us"] else None,
                   "yield_us_p99": round(pct(r["yield_us"], .99) / 1e3, 2) if r["yield_us"] else None,
                   "drain_us_p50": round(pct(r["drain_us"], .5) / 1e3, 2) if r["drain_us"] else None,
                   "drain_us_p99": round(pct(r["drain_us"], .99) / 1e3, 2) if r["drain_us"] else None,
                   "grant_us_p50": round(pct(r["grant_us"], .5) / 1e3, 2) if r["grant_us"] else None,
                   "grant_us_p99": round(pct(r["grant_us"], .99) / 1e3, 2) if r["grant_us"] else None,
                   "lost_throughput": round(lost, 4)}
            res["sweep"].append(row)
            print(json.dumps(row), flush=True)
    # host -> device control latency: host write -> device install, acknowledged
    # into host memory (round trip on the host clock; one way <= RTT)
    rtt = [x / 1e3 for x in dom.ctl_roundtrip(200)]
    res["host_device_ctl_roundtrip_us"] = {"p50": round(pct(rtt, .5), 2), "p90": round(pct(rtt, .9), 2),
                                           "p99": round(pct(rtt, .99), 2), "n": len(rtt)}
    print(json.dumps(res["host_device_ctl_roundtrip_us"]))
    dom.stop(); dom.close()
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(res, open("gpurun_out/migration_sweep.json", "w"), indent=1)

if __name__ == "__main__":
    main()
