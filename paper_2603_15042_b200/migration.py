"""SM-quota migration measurement (BASELINE config 3).

A tenant's launch runs while the executor's device-timer program flips its
quota between two control words (all SMs <-> a quarter of them) every P us,
with no host round trip.  From the device logs (switch log, control log):
  * yield latency per revoked SM: first switch-away after a flip - flip time
    (an SM leaves only at a logical-block boundary, so <= one block);
  * drain: the SM's second lane leaving;
  * grant latency: first block of the tenant on a regained SM - flip time;
  * lost throughput: 1 - achieved blocks/s / (unflipped blocks/s x time-weighted SM fraction).
Reference: signal_preempt / next_boundary_work / on_preempt_boundary
(src/engine/engine.cpp:756-806,16-24,925-984) and the PreemptionRecord
boundary_wait it measures (include/corosim/runtime/migration.hpp:47-53).
"""
from __future__ import annotations

import numpy as np

from . import _abi


def pct(v, q):
    v = sorted(v)
    return v[min(len(v) - 1, int(q * len(v)))] if v else None

def spin_kernel(dom, block_us, nblocks):
    """A stream of fixed-length logical blocks (test body)."""
    import torch
    # torch.empty: no fill kernel (nothing but copies may run beside the resident executor)
    out = torch.empty(3 * nblocks, dtype=torch.int64, device=f"cuda:{dom.device}")
    kid = dom.kernel(f"spin/{block_us}us", _abi.BODY_SPIN, (nblocks, 1, 1), _abi.SpinArgs(out.data_ptr(), int(block_us * 1000)))
    dom._args_keep.append(out)
    return kid


def run(dom, t, kid, period_us):
    """One launch of `kid` while the device timer flips tenant t's quota
    between all SMs and a quarter of them every period_us (0: no flips)."""
    n = dom.num_sms
    full = dom.mask(t, 0, n)
    quarter = dom.mask(t, 0, n // 4)
    dom.poll(1 << 16)
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
    return {"blocks_per_s": c.grid / span, "span_s": span, "flips": len(flips), "yield_us": yields,
            "sm_fraction": sm_fraction,
            "drain_us": drains, "grant_us": grants}


def summarize(r, unflipped_bps):
    """p50/p99 latencies (us) and lost throughput of one sweep point."""
    f = lambda v, q: round(pct(v, q) / 1e3, 2) if v else None  # noqa: E731
    return {"flips": r["flips"], "yield_us_p50": f(r["yield_us"], .5), "yield_us_p99": f(r["yield_us"], .99),
            "drain_us_p50": f(r["drain_us"], .5), "drain_us_p99": f(r["drain_us"], .99),
            "grant_us_p50": f(r["grant_us"], .5), "grant_us_p99": f(r["grant_us"], .99),
            "lost_throughput": round(1.0 - r["blocks_per_s"] / (unflipped_bps * r["sm_fraction"]), 4)}
