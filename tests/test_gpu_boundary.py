"""The drop-in boundary on a B200: user policies injected through
the C-ABI vtable (SimEngine(Scenario, std::unique_ptr<Policy>), engine.hpp:155)
with the reference's fail-safe validation (apply_decision, engine.cpp:688-754:
illegal -> Defer + policy_errors, incl. the quarantined-vctx Remap check at
engine.cpp:726-728), ds_snapshot, kernel-record immutability (types.cpp:39-48,
engine.cpp:1379-1383), the device-measured overhead ledger (engine.hpp:94-107),
bind errors, and the C++ façade's GPU half."""
import os
import subprocess
import time
from fractions import Fraction

import pytest
import torch

from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200 import migration as mg
from paper_2603_15042_b200.runtime import Domain, Engine, UserPolicy

pytestmark = pytest.mark.gpu

TIERS = [Fraction(1, 4), Fraction(1, 2), Fraction(1)]


def test_facade_gpu(tmp_path):
    from test_facade import build_facade_test
    exe = build_facade_test(tmp_path / "test_facade")
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "gpu facade tests: ok" in r.stdout


class Adversarial(UserPolicy):
    """the first `bad` decisions Remap to a bound pctx (or to no
    pctx); then the smallest free feasible tier, or Direct when bound."""
    name = "adversarial"

    def __init__(self, bad):
        self.bad, self.calls = bad, 0

    def on_launch(self, view, launch):
        self.calls += 1
        if self.calls <= self.bad:
            bound = [p.id for p in view.pctxs if p.bound is not None and p.bound != launch.vctx]
            return (_abi.DISPATCH_REMAP, bound[0] if bound else 999)
        v = next(x for x in view.vctxs if x.id == launch.vctx)
        if v.bound:
            return (_abi.DISPATCH_DIRECT, -1)
        free = [p for p in view.pctxs if p.bound is None and p.available and
                view.bound_tier_sums[p.device] + p.tier <= 1]
        return (_abi.DISPATCH_REMAP, min(free, key=lambda p: p.tier).id) if free else (_abi.DISPATCH_DEFER, -1)


def _spin(dom, ns, grid=296, name="spin"):
    out = torch.zeros(3 * grid, dtype=torch.int64, device="cuda")
    k = dom.kernel(name, _abi.BODY_SPIN, (grid, 1, 1), _abi.SpinArgs(out.data_ptr(), ns))
    return k, out


def test_user_policy_illegal_decisions_defer_with_policy_errors():
    with Domain(0, tiers=TIERS, block_log_capacity=0) as dom:
        t0 = dom.tenant("decode", _abi.LATENCY_CRITICAL)
        t1 = dom.tenant("train", _abi.BEST_EFFORT)
        ks, _ = _spin(dom, 20_000)
        dom.start()
        pol = Adversarial(bad=5)
        eng = Engine(dom, policy=pol)
        j0 = eng.add_job(t0, _abi.LATENCY_CRITICAL)
        j1 = eng.add_job(t1, _abi.BEST_EFFORT)
        eng.start()
        try:
            recs = [eng.submit(j, [ks, ks], "spin", phase=_abi.DECODE if j == j0 else _abi.TRAINING, grid_size=296,
                               base_hint_ns=100_000, saturation=Fraction(1, 2)) for j in (j0, j1) for _ in range(3)]
            for r in recs:
                eng.wait(r, 30000)
            snap = eng.snapshot()
            ctr = eng.counters()
        finally:
            eng.stop()
            eng.close()
    assert ctr["policy_errors"] == 5, ctr
    assert ctr["completed"] == 6
    assert [p.tier for p in snap.pctxs] == TIERS
    assert [v.id for v in snap.vctxs] == [0, 1]


class QuarantineProbe(UserPolicy):
    """Remaps a quarantined vctx to the full tier once (illegal: a quarantined
    vctx may bind only the pool's minimal tier, engine.cpp:726-728), then to
    the minimal tier; unquarantined vctxs go to the full tier."""
    name = "quarantine-probe"

    def __init__(self):
        self.tried_big = False

    def on_launch(self, view, launch):
        v = next(x for x in view.vctxs if x.id == launch.vctx)
        if v.bound:
            return (_abi.DISPATCH_DIRECT, -1)
        free = sorted((p for p in view.pctxs if p.bound is None and p.available), key=lambda p: p.tier)
        if not free:
            return (_abi.DISPATCH_DEFER, -1)
        if v.quarantined and not self.tried_big:
            self.tried_big = True
            return (_abi.DISPATCH_REMAP, free[-1].id)
        return (_abi.DISPATCH_REMAP, (free[0] if v.quarantined else free[-1]).id)


def test_quarantined_vctx_remap_above_min_tier_is_a_policy_error():
    with Domain(0, tiers=TIERS, block_log_capacity=0) as dom:
        t0 = dom.tenant("hung", _abi.BEST_EFFORT)
        # 296 blocks x 300 us on the full tier: ~300 us, >> 3 x the 20 us hint
        ks, _ = _spin(dom, 300_000, grid=296 * 4)
        dom.start()
        pol = QuarantineProbe()
        eng = Engine(dom, policy=pol, hang_detection=True, hang_threshold=3.0)
        j0 = eng.add_job(t0, _abi.BEST_EFFORT)
        eng.start()
        try:
            r = eng.submit(j0, [ks], "spin", phase=_abi.TRAINING, grid_size=296 * 4, base_hint_ns=20_000)
            eng.wait(r, 60000)
            ctr = eng.counters()
            rec = eng.record(r)
        finally:
            eng.stop()
            eng.close()
    assert pol.tried_big
    assert ctr["policy_errors"] >= 1, ctr
    assert rec.state == 2 and rec.preempted >= 1


def test_kernel_record_mutation_is_detected():
    """A body that writes into another kernel's immutable argument block (here
    a spin kernel whose output pointer aims at it) is caught by the
    fingerprint check, by ds_verify_kernels and at engine finalize."""
    with Domain(0, tiers=[Fraction(1)], block_log_capacity=0) as dom:
        t = dom.tenant("t", _abi.BEST_EFFORT)
        kb, _ = _spin(dom, 1000, grid=4, name="victim")
        info = dom.kernel_info(kb)
        ka = dom.kernel("mutator", _abi.BODY_SPIN, (1, 1, 1), _abi.SpinArgs(info.args_device, 1000))
        dom.start()
        assert dom.verify_kernels() == -1
        eng = Engine(dom, policy="static", assignments={0: 0})
        try:
            j = eng.add_job(t, _abi.BEST_EFFORT)
            eng.start()
            r = eng.submit(j, [ka], "mutator", grid_size=1)
            fp0 = eng.job_fingerprint(j)
            assert fp0 != 0
            eng.wait(r, 30000)
            assert eng.job_fingerprint(j) == fp0
            assert dom.verify_kernels() == kb
            with pytest.raises(_abi.DsError) as ei:
                eng.stop()
            assert ei.value.code == _abi.RECORD_MUTATED
        finally:
            eng.close()


def test_ledger_from_device_timestamps():
    """Quota flips 100% <-> 25% between two spin tenants every 200 us: the
    device ledger sees lane yields (boundary waits no longer than a block plus
    the install), grants and switches."""
    with Domain(0, tiers=[Fraction(1)], block_log_capacity=0, lend_idle_sms=False) as dom:
        a = dom.tenant("a", _abi.BEST_EFFORT)
        b = dom.tenant("b", _abi.BEST_EFFORT)
        ka, _ = _spin(dom, 10_000, grid=296 * 40, name="a")
        kb, _ = _spin(dom, 10_000, grid=296 * 40, name="b")
        dom.start()
        n = dom.num_sms
        wa = [a if i < n else b for i in range(n)]
        wb = [a if i < n // 4 else b for i in range(n)]
        l0 = dom.ledger()
        dom.quota_periodic(200_000, wa, wb)
        sa, sb = dom.launch(a, ka), dom.launch(b, kb)
        dom.wait(a, sa, 60000)
        dom.wait(b, sb, 60000)
        dom.quota_periodic(0, wa, wa)
        l1 = dom.ledger()
    d = {k: l1[k] - l0[k] for k in l1}
    print(d)
    assert d["preemptions"] > 100 and d["migrations"] > 100 and d["ctx_switches"] > 100
    assert d["preempt_total_ns"] / d["preemptions"] < 40_000      # a 10 us block + install skew
    assert d["migration_total_ns"] / d["migrations"] < 60_000
