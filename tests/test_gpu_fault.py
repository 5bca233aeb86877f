"""Fault containment (reference on_hang_check,
engine.cpp:542-561,1011-1035) and the JSONL event log (engine.cpp:316-329):
a soft-hung record (running > threshold x prediction) quarantines its vctx,
its SMs yield at a logical-block boundary, and it resumes — never restarts —
confined to the pool's minimum tier."""
from fractions import Fraction

import pytest
import torch

from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain, Engine

pytestmark = pytest.mark.gpu

REF_KINDS = {"Arrival", "LaunchReady", "KernelStart", "KernelFinish", "PreemptSignal", "MigrationDone",
             "FaultInjected", "HangCheck"}


def test_soft_hang_is_quarantined_to_min_tier():
    out = torch.zeros(4096 * 4, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    tiers = [Fraction(1, 4), Fraction(1, 2), Fraction(1)]
    with Domain(0, tiers=tiers, block_log_capacity=0) as dom:
        dom.start()
        t = dom.tenant("maybe-hung", _abi.BEST_EFFORT)
        normal = dom.kernel("spin", _abi.BODY_SPIN, (600, 1, 1), _abi.SpinArgs(out.data_ptr(), 20_000))
        hung = dom.kernel("spin", _abi.BODY_SPIN, (600, 1, 1), _abi.SpinArgs(out.data_ptr(), 400_000))
        eng = Engine(dom, policy="slo-aware", hang_detection=True, hang_threshold=3.0, capture_log=True)
        j = eng.add_job(t, _abi.BEST_EFFORT)
        eng.start()
        try:
            recs = [eng.submit(j, [normal], "spin", grid_size=600, base_hint_ns=100_000) for _ in range(4)]
            for r in recs:
                eng.wait(r, 30000)
            assert eng.quarantines() == []
            bad = eng.submit(j, [hung], "spin", grid_size=600, base_hint_ns=100_000)  # same signature: ~20x slower
            eng.wait(bad, 60000)
            after = eng.submit(j, [normal], "spin", grid_size=600)
            eng.wait(after, 30000)
            q = eng.quarantines()
            log = eng.event_log()
            info_bad, info_after = eng.record(bad), eng.record(after)
        finally:
            eng.stop()
            eng.close()
    assert [x[0] for x in q] == [j]
    assert info_bad.preempted >= 1                     # its SMs were revoked mid-kernel ...
    assert dom.tiers[info_bad.pctx] == Fraction(1, 4)  # ... and it finished on the minimum tier
    assert dom.tiers[info_after.pctx] == Fraction(1, 4)
    kinds = [e["kind"] for e in log]
    assert set(kinds) <= REF_KINDS
    assert kinds.count("Arrival") == 6 and kinds.count("KernelFinish") == 6
    assert kinds.count("HangCheck") == 1
    hc = next(e for e in log if e["kind"] == "HangCheck")
    assert hc["flagged"] is True and hc["vctx"] == j
    seqs = [e["seq"] for e in log]
    assert seqs == sorted(seqs) and len(set(seqs)) == len(seqs)
