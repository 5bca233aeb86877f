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

from paper_2603_15042_b200.migration import pct, run as run_kernel, spin_kernel


def run(dom, t, block_us, period_us, nblocks):
    return run_kernel(dom, t, spin_kernel(dom, block_us, nblocks), period_us)


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
