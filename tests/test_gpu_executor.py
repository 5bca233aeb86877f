"""GPU parity of the coroutine executor (run on a B200 via gpurun).

The reduction tenant is the one direct bit-exact bridge to the reference
(reduction_result, src/numlab/equivalence.cpp:19-25): its result must equal
the reference's bits (tests/golden/reduction_golden.json, generated from the
reference library) both solo and as a coroutine whose SM quota changes
mid-kernel; the atomizing mutant (engine.hpp:68-71) must diverge."""
import ctypes
import json
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

from oracle import loader, numlab as nl
from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain, solo_launch

pytestmark = pytest.mark.gpu


def dfull(n, value, dtype):
    """Device buffer filled by a host->device copy (copy engine only: no
    kernel, so it is safe while the persistent executor is resident)."""
    return torch.from_numpy(np.full(n, value, dtype=dtype)).cuda()

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reduction_golden.json")))
FMT = {"fp16": 0, "bf16": 1, "fp32": 2}


def seeded_tensor(seed, n, fmt):
    cn = loader.cnumlab()
    bits = (ctypes.c_uint32 * max(n, 1))()
    cn.cn_seeded_bits(seed, n, FMT[fmt], bits)
    a = np.frombuffer(bits, dtype=np.uint32)[:n]
    if fmt == "fp32":
        return torch.from_numpy(a.astype(np.uint32).view(np.int32).copy()).cuda()
    return torch.from_numpy(a.astype(np.uint16).view(np.int16).copy()).cuda()


class ReduceKernel:
    def __init__(self, seed, n, fmt, grid):
        self.x = seeded_tensor(seed, n, fmt) if n > 0 else dfull(1, 0, np.int32)
        self.partials = dfull(max(grid, 1), 0, np.int32)
        self.out = dfull(1, -1, np.int32)
        self.ticket = dfull(1, 0, np.int32)
        self.args = _abi.ReduceArgs(self.x.data_ptr(), self.partials.data_ptr(), self.out.data_ptr(),
                                    self.ticket.data_ptr(), n, FMT[fmt], 1)
        self.grid = grid

    def result(self):
        # .item() syncs only torch's stream; never device-synchronize while
        # the persistent executor is resident
        return int(self.out.item()) & 0xFFFFFFFF


def test_solo_reduction_matches_reference_golden():
    for c in GOLDEN["cases"]:
        n = c.get("n", GOLDEN["n"])
        k = ReduceKernel(c["seed"], n, c["fmt"], c["grid"])
        solo_launch(0, "reduce", _abi.BODY_REDUCE_CHUNKS, (c["grid"], 1, 1), k.args)
        assert k.result() == c["bits"], c


@pytest.fixture
def dom():
    """Domain created but not started: solo baselines run first, on an
    otherwise idle GPU; tests call dom.start() themselves."""
    d = Domain(0, tiers=[Fraction(1, 4), Fraction(1, 2), Fraction(1)], block_log_capacity=1 << 20)
    yield d
    d.stop()
    d.close()


def test_coroutine_reduction_with_quota_flips_is_bit_exact(dom):
    dom.start()
    t = dom.tenant("lab", _abi.BEST_EFFORT)
    full = dom.mask(t, 0, dom.num_sms)
    quarter = dom.mask(t, 0, dom.num_sms // 4)
    few = dom.mask(t, 5, 3)
    dom.quota_set(full)
    cases = [c for c in GOLDEN["cases"] if c["grid"] in (7, 37, 64, 148) and c["seed"] < 4]
    kernels = []
    for i, c in enumerate(cases):
        k = ReduceKernel(c["seed"], c.get("n", GOLDEN["n"]), c["fmt"], c["grid"])
        kid = dom.kernel(f"reduce/{c['fmt']}", _abi.BODY_REDUCE_CHUNKS, (c["grid"], 1, 1), k.args)
        kernels.append((c, k, kid))
    # device-side quota changes at exact claim counts of launch 0 and 1
    dom.quota_at_claim(t, 0, 3, quarter)
    dom.quota_at_claim(t, 1, 2, few)
    dom.quota_at_claim(t, 2, 1, full)
    last = None
    for c, k, kid in kernels:
        last = dom.launch(t, kid)
    dom.wait(t, last)
    for c, k, kid in kernels:
        assert k.result() == c["bits"], c
    # transcript = launch configs in program order, unchanged
    assert dom.transcript(t) == [(kid, c["grid"]) for c, k, kid in kernels]
    assert dom.logical_progress(t) == len(kernels)
    # every logical block claimed exactly once
    log = dom.block_log()
    for seq, (c, k, kid) in enumerate(kernels):
        blocks = sorted(r.block for r in log if r.tenant == t and r.seq == seq)
        assert blocks == list(range(c["grid"])), seq
    # the triggers fired (control changed on the device)
    assert len([r for r in dom.ctl_log() if r.source == 1]) == 3


def test_atomizing_mutant_breaks_equivalence(dom):
    dom.start()
    t = dom.tenant("lab", _abi.BEST_EFFORT)
    dom.quota_set(dom.mask(t, 0, dom.num_sms))
    diverged = 0
    for seed in range(6):
        want = next(c for c in GOLDEN["cases"] if c["fmt"] == "fp16" and c["seed"] == seed and c["grid"] == 64)
        k = ReduceKernel(seed, 4096, "fp16", 64)
        kid = dom.kernel("reduce/fp16", _abi.BODY_REDUCE_CHUNKS, (64, 1, 1), k.args)
        s = dom.launch_atomized(t, kid, Fraction(1, 4))
        dom.wait(t, s)
        assert dom.transcript(t)[-1] == (kid, 16)  # executed grid rewritten to floor(64/4)
        ref16 = loader.cnumlab().cn_reduction_result(seed, 4096, 0, 16)
        assert k.result() == ref16
        diverged += k.result() != want["bits"]
    assert diverged >= 4


def sgemm_inputs(M, N, K):
    cn = loader.cnumlab()
    A = (ctypes.c_float * (M * K))()
    B = (ctypes.c_float * (K * N))()
    cn.cn_uniform_f32(1, M * K, -1.0, 1.0, A)
    cn.cn_uniform_f32(2, K * N, -1.0, 1.0, B)
    return (np.frombuffer(A, dtype=np.float32).reshape(M, K).copy(),
            np.frombuffer(B, dtype=np.float32).reshape(K, N).copy())


def test_sgemm_coroutine_mid_kernel_quota_change_bit_exact(dom):
    """BASELINE config 1: SGEMM 1024^3 as one coroutine, quota 100% -> 25% at
    30% of claimed blocks -> 100% at 60%; bit-exact vs solo and vs the CPU
    k-ascending fma oracle."""
    M = N = K = 1024
    A, B = sgemm_inputs(M, N, K)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    C_solo = torch.zeros(M, N, device="cuda")
    C_co = torch.zeros(M, N, device="cuda")
    a_solo = _abi.SgemmArgs(dA.data_ptr(), dB.data_ptr(), C_solo.data_ptr(), M, N, K, 0)
    a_co = _abi.SgemmArgs(dA.data_ptr(), dB.data_ptr(), C_co.data_ptr(), M, N, K, 0)
    grid = (N // 64, M // 64, 1)
    solo_launch(0, "sgemm", _abi.BODY_SGEMM, grid, a_solo)
    torch.cuda.synchronize()
    dom.start()
    t = dom.tenant("sgemm", _abi.BEST_EFFORT)
    dom.quota_set(dom.mask(t, 0, dom.num_sms))
    kid = dom.kernel("sgemm", _abi.BODY_SGEMM, grid, a_co)
    nblk = grid[0] * grid[1]
    dom.quota_at_claim(t, 0, int(0.3 * nblk), dom.mask(t, 0, dom.num_sms // 4))
    dom.quota_at_claim(t, 0, int(0.6 * nblk), dom.mask(t, 0, dom.num_sms))
    s = dom.launch(t, kid)
    dom.wait(t, s)
    # host-side comparison: torch kernels cannot co-reside with the executor
    # (its CTAs pin the SM shared-memory carveout), copies can
    got = C_co.cpu().numpy()
    assert np.array_equal(C_solo.cpu().numpy().view(np.uint32), got.view(np.uint32))
    # CPU fma-chain oracle on a sample of rows
    cn = loader.cnumlab()
    rows = [0, 1, 511, 1023]
    Cref = np.zeros((M, N), dtype=np.float32)
    Ap = A.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
    Bp = B.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
    Cp = Cref.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
    for r in rows:
        cn.cn_sgemm_fma(Ap, Bp, Cp, M, N, K, r, r + 1)
    for r in rows:
        assert np.array_equal(got[r].view(np.uint32), Cref[r].view(np.uint32)), r
    # blocks ran on the quarter set while the 25% quota was in force
    log = [b for b in dom.block_log() if b.tenant == t]
    assert sorted(b.block for b in log) == list(range(nblk))


def test_spin_arbiter_two_tenants_disjoint_sets(dom):
    """Two tenants with disjoint SM sets never share an SM; a quota change
    moves SMs between them at block boundaries only."""
    dom.start()
    n = dom.num_sms
    a = dom.tenant("a", _abi.LATENCY_CRITICAL)
    b = dom.tenant("b", _abi.BEST_EFFORT)
    owner = [a if i < n // 2 else b for i in range(n)]
    dom.quota_set(owner)
    outa = dfull(3 * 2000, 0, np.int64)
    outb = dfull(3 * 2000, 0, np.int64)
    ka = dom.kernel("spin/a", _abi.BODY_SPIN, (2000, 1, 1), _abi.SpinArgs(outa.data_ptr(), 20000))
    kb = dom.kernel("spin/b", _abi.BODY_SPIN, (2000, 1, 1), _abi.SpinArgs(outb.data_ptr(), 20000))
    sa = dom.launch(a, ka)
    sb = dom.launch(b, kb)
    dom.wait(a, sa)
    dom.wait(b, sb)
    smids = dom.smids()
    a_sms = {smids[i] for i in range(n // 2)}
    ra = outa.view(-1, 3).cpu().numpy()
    rb = outb.view(-1, 3).cpu().numpy()
    assert set(ra[:, 0].tolist()) <= a_sms
    assert not (set(rb[:, 0].tolist()) & a_sms)
    sw = dom.switch_log()
    assert len(sw) >= n  # every SM switched from idle to its tenant at least once
