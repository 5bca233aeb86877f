"""Local exceptions (reference apply_local_exception,
engine.cpp:1049-1083, FaultSpec::LocalException engine.hpp:21-28).

A tenant that faults fails alone: the device stops handing out its blocks,
blocks already running finish (their in-launch waits give up), its launches
never complete and later launches are refused (arrivals of a failed vctx are
dropped, engine.cpp:810-819).  The co-located tenant keeps its SMs' results
bit-identical to its solo run, and the executor keeps serving."""
import time
from fractions import Fraction

import numpy as np
import pytest
import torch

from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200._abi import DsError
from paper_2603_15042_b200.runtime import Domain, Engine
from paper_2603_15042_b200.tenants import DecodeConfig, DecodeModel
from gpu_util import sgemm_copies as _sgemm

pytestmark = pytest.mark.gpu


def test_injected_fault_mid_decode_leaves_training_bit_exact():
    m = DecodeModel(DecodeConfig(layers=2, vocab=2048, L=96, attn_splits=2), seed=5)
    keep, sargs, grid = _sgemm(copies=4)
    Cs = keep[2]
    torch.cuda.synchronize()
    with Domain(0, tiers=[Fraction(1, 2), Fraction(1)], block_log_capacity=1 << 20) as dom:
        dom.start()
        td = dom.tenant("decode", _abi.LATENCY_CRITICAL)
        ts = dom.tenant("train", _abi.BEST_EFFORT)
        n = dom.num_sms
        dom.quota_set([td if i < n // 2 else ts for i in range(n)])
        kids = m.register(dom)
        ks = [dom.kernel("sgemm", _abi.BODY_SGEMM, grid, a) for a in sargs[1:]]
        # a long chain of decode steps (split-K GEMVs, attention, argmax) ...
        last_d = None
        for _ in range(40):
            for k in kids:
                last_d = dom.launch(td, k)
        # ... next to four training launches
        seqs = [dom.launch(ts, k) for k in ks]
        time.sleep(0.003)
        dom.fault_inject(td)  # lands while decode blocks are in flight
        f = dom.tenant_fault(td)
        for s in seqs:
            dom.wait(ts, s, 60000)
        with pytest.raises(DsError) as ei:
            dom.wait(td, last_d, 10000)
        assert ei.value.code == _abi.TENANT_FAILED
        with pytest.raises(DsError) as ei:
            dom.launch(td, kids[0])
        assert ei.value.code == _abi.TENANT_FAILED
        # the executor still serves: the failed tenant's SMs go to training
        dom.quota_set([ts] * n)
        s = dom.launch(ts, ks[0])
        dom.wait(ts, s, 60000)
        got = [C.cpu() for C in Cs]
        blog = dom.block_log()
        prog = dom.logical_progress(td)
    assert f is not None and f["code"] == _abi.FAULT_INJECTED and f["block"] == 0xFFFFFFFF
    assert 0 < f["first_failed"] <= prog        # launches before it had finished intact
    assert 0 < prog < 40 * len(kids)            # it died mid-chain
    ref = got[0].numpy().view(np.uint32)
    for C in got[1:]:
        assert np.array_equal(C.numpy().view(np.uint32), ref)
    # no decode block starts after the kill (allowing the blocks claimed just
    # before it a few microseconds to reach their body)
    late = [b for b in blog if b.tenant == td and b.t_start > f["t"] + 50_000]
    assert late == []


def test_bad_token_raises_local_exception_in_the_embed_body():
    d, vocab = 4096, 1000
    g = torch.Generator(device="cuda").manual_seed(3)
    table = (torch.rand(vocab, d, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    tokens = torch.arange(32, dtype=torch.int32, device="cuda")
    tokens[7] = vocab + 3
    h = torch.zeros(32, d, dtype=torch.bfloat16, device="cuda")
    spin_out = torch.zeros(3 * 400, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    with Domain(0, tiers=[Fraction(1)], block_log_capacity=0) as dom:
        dom.start()
        te = dom.tenant("decode", _abi.LATENCY_CRITICAL)
        tsp = dom.tenant("other", _abi.BEST_EFFORT)
        n = dom.num_sms
        dom.quota_set([te if i % 2 else tsp for i in range(n)])
        ke = dom.kernel("embed", _abi.BODY_EMBED, (32, 1, 1),
                        _abi.EmbedArgs(table.data_ptr(), tokens.data_ptr(), h.data_ptr(), d, vocab, 0))
        kspin = dom.kernel("spin", _abi.BODY_SPIN, (400, 1, 1), _abi.SpinArgs(spin_out.data_ptr(), 20_000))
        ss = dom.launch(tsp, kspin)
        se = dom.launch(te, ke)
        with pytest.raises(DsError) as ei:
            dom.wait(te, se, 10000)
        assert ei.value.code == _abi.TENANT_FAILED
        dom.wait(tsp, ss, 30000)
        s2 = dom.launch(tsp, kspin)
        dom.wait(tsp, s2, 30000)
        f = dom.tenant_fault(te)
        assert dom.tenant_fault(tsp) is None
    assert f["code"] == _abi.FAULT_BAD_INPUT and f["seq"] == se and f["block"] == 7
    assert f["first_failed"] == se
    rows = h.cpu()
    for b in (0, 1, 31):  # the valid rows were still gathered
        assert torch.equal(rows[b], table[b].cpu())


def test_engine_local_exception_fails_the_bound_job_only():
    keep, sargs, grid = _sgemm(copies=3)
    Cs = keep[2]
    spin_out = torch.zeros(3 * 300, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    tiers = [Fraction(1, 4), Fraction(1, 2), Fraction(3, 4), Fraction(1)]
    with Domain(0, tiers=tiers, block_log_capacity=0) as dom:
        dom.start()
        td = dom.tenant("decode", _abi.LATENCY_CRITICAL)
        ts = dom.tenant("train", _abi.BEST_EFFORT)
        kspin = dom.kernel("decode/spin", _abi.BODY_SPIN, (300, 1, 1), _abi.SpinArgs(spin_out.data_ptr(), 30_000))
        ks = [dom.kernel("train/sgemm", _abi.BODY_SGEMM, grid, a) for a in sargs[1:]]
        eng = Engine(dom, policy="tpot-first", capture_log=True, reset_delay_ns=500_000)
        jd = eng.add_job(td, _abi.LATENCY_CRITICAL)
        js = eng.add_job(ts, _abi.BEST_EFFORT)
        eng.start()
        try:
            # nothing bound yet: a fault on pctx 0 has no effect (engine.cpp:1051-1058)
            eng.fault_local(0)
            tr = [eng.submit(js, [k], "train/sgemm", phase=_abi.TRAINING, grid_size=256) for k in ks]
            dr = [eng.submit(jd, [kspin] * 4, "decode/spin", phase=_abi.DECODE, grid_size=300, tpot_ns=50_000_000)
                  for _ in range(50)]
            eng.wait(dr[0], 30000)
            p = None
            for _ in range(2000):
                p = dom.bound_pctx(td)
                if p >= 0:
                    break
                time.sleep(0.0005)
            assert p is not None and p >= 0
            eng.fault_local(p)
            assert eng.job_status(jd) == _abi.FAILED
            assert eng.job_status(js) == _abi.ACTIVE
            with pytest.raises(DsError) as ei:
                eng.wait(dr[-1], 10000)
            assert ei.value.code == _abi.TENANT_FAILED
            with pytest.raises(DsError):
                eng.submit(jd, [kspin], "decode/spin", phase=_abi.DECODE, grid_size=300)
            for r in tr:
                eng.wait(r, 60000)
            info = eng.record(dr[-1])
            log = eng.event_log()
            ctr = eng.counters()
        finally:
            eng.stop()
            eng.close()
        got = [C.cpu() for C in Cs]
    assert info.state == 3
    assert ctr["failed_jobs"] == 1
    faults = [e for e in log if e["kind"] == "FaultInjected"]
    assert faults[0]["fault"] == "local" and faults[0]["effect"] == "none"
    assert faults[1]["vctx"] == jd and faults[1]["pctx"] == p
    ref = got[0].numpy().view(np.uint32)
    for C in got[1:]:
        assert np.array_equal(C.numpy().view(np.uint32), ref)

