"""Sub-block yields (ds_tenant_abandonable + GemmArgs.abandon): a tcgen05
GEMM tile gives its logical block up within one k-block when its SM is
revoked and re-runs from scratch later.  The result stays bit-identical to
the solo GEMM, every block retires exactly once, and the yield latency drops
from a whole tile (~100 us) to a few microseconds."""
from fractions import Fraction

import numpy as np
import pytest
import torch

from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200 import migration as mg
from paper_2603_15042_b200.runtime import Domain, solo_launch

pytestmark = pytest.mark.gpu

M, N, K = 4096, 4096, 8192


def _operands():
    g = torch.Generator(device="cuda").manual_seed(7)
    A = ((torch.rand(M, K, device="cuda", generator=g) * 2 - 1)).to(torch.bfloat16)
    B = ((torch.rand(N, K, device="cuda", generator=g) * 2 - 1)).to(torch.bfloat16)
    return A, B


@pytest.mark.parametrize("abandon", [1, 2, 0])
def test_gemm_tiles_abandon_on_revocation_bit_exact(abandon):
    A, B = _operands()
    C_solo = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    C_co = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    a_solo = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C_solo.data_ptr(), M, N, K, group_m=16)
    a_co = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C_co.data_ptr(), M, N, K, group_m=16, abandon=abandon)
    grid = _abi.gemm_grid(M, N)
    solo_launch(0, "gemm", _abi.BODY_GEMM_BF16, grid, a_solo)
    torch.cuda.synchronize()
    with Domain(0, tiers=[Fraction(1)], block_log_capacity=1 << 18) as dom:
        t = dom.tenant("train", _abi.BEST_EFFORT)
        if abandon:
            dom.set_abandonable(t)
        kid = dom.kernel("train/gemm", _abi.BODY_GEMM_BF16, grid, a_co)
        dom.start()
        # quota 100% <-> 25% by the device timer: every 50 us with abandoning
        # (many revocations per tile), every 100 us without (a tile is ~100 us)
        r = mg.run(dom, t, kid, 50 if abandon else 100)
        blog = [b for b in dom.block_log() if b.tenant == t]
        got = C_co.cpu()
    assert np.array_equal(got.view(torch.int16).numpy(), C_solo.cpu().view(torch.int16).numpy())
    done = sorted(b.block for b in blog if b.flags == 0)
    assert done == list(range(grid[0]))           # every tile retired exactly once
    gave_up = [b for b in blog if b.flags == 1]
    y = sorted(r["yield_us"])
    p50 = y[len(y) // 2] / 1e3 if y else None
    print(f"abandon={abandon}: flips {r['flips']}, abandoned attempts {len(gave_up)}, yield p50 {p50} us")
    if abandon == 2:
        assert len(gave_up) > 0   # spilled and resumed: slower yield (the spill), no lost work
    elif abandon:
        assert len(gave_up) > 0
        # measured p50 ~7 us, p99 ~9 us (bench config 3 reports them); the
        # assert only pins "well under a whole ~120 us tile" so clock and
        # power-cap variation cannot make it flaky
        assert p50 < 50.0
    else:
        assert gave_up == []


@pytest.mark.parametrize("mode", [1, 2])
def test_abandon_across_back_to_back_launches(mode):
    """Several launches enqueued back to back while tiles are abandoned
    (an abandonable tenant opens launch s+1 only once s completed, so no lane
    parks on s+1 while s's tiles wait in the retry ring): nothing deadlocks,
    every (launch, tile) retires exactly once and the output stays bit-exact."""
    A, B = _operands()
    C_solo = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    C_co = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    a_solo = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C_solo.data_ptr(), M, N, K, group_m=16)
    a_co = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C_co.data_ptr(), M, N, K, group_m=16, abandon=mode)
    grid = _abi.gemm_grid(M, N)
    solo_launch(0, "gemm", _abi.BODY_GEMM_BF16, grid, a_solo)
    torch.cuda.synchronize()
    with Domain(0, tiers=[Fraction(1)], block_log_capacity=1 << 20) as dom:
        t = dom.tenant("train", _abi.BEST_EFFORT)
        dom.set_abandonable(t)
        kid = dom.kernel("train/gemm", _abi.BODY_GEMM_BF16, grid, a_co)
        dom.start()
        n = dom.num_sms
        full, eighth = dom.mask(t, 0, n), dom.mask(t, 0, n // 8)
        dom.quota_set(full)
        dom.clear_logs()
        dom.quota_periodic(40_000, full, eighth)  # 100% <-> 1/8 every 40 us
        seqs = [dom.launch(t, kid) for _ in range(4)]
        dom.wait(t, seqs[-1], 120000)
        dom.quota_periodic(0, full, full)
        blog = [b for b in dom.block_log() if b.tenant == t]
        got = C_co.cpu()
    assert np.array_equal(got.view(torch.int16).numpy(), C_solo.cpu().view(torch.int16).numpy())
    for s in seqs:
        done = sorted(b.block for b in blog if b.flags == 0 and b.seq == s)
        assert done == list(range(grid[0])), s
    assert sum(b.flags == 1 for b in blog) > 0


@pytest.mark.parametrize("mode", [1, 2])
def test_engine_decode_preempts_abandonable_training(mode):
    """TPOT-First engine: latency-critical records bind SMs that training
    tiles hold; abandonable tiles give them up mid-tile and re-run, training
    output stays bit-exact."""
    from paper_2603_15042_b200.runtime import Engine
    A, B = _operands()
    C_solo = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    C_co = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    a_solo = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C_solo.data_ptr(), M, N, K, group_m=16)
    a_co = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C_co.data_ptr(), M, N, K, group_m=16, abandon=mode)
    grid = _abi.gemm_grid(M, N)
    solo_launch(0, "gemm", _abi.BODY_GEMM_BF16, grid, a_solo)
    spin_out = torch.zeros(3 * 600, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    tiers = [Fraction(1, 4), Fraction(1, 2), Fraction(3, 4), Fraction(1)]
    with Domain(0, tiers=tiers, block_log_capacity=1 << 20) as dom:
        td = dom.tenant("decode", _abi.LATENCY_CRITICAL)
        tt = dom.tenant("train", _abi.BEST_EFFORT)
        dom.set_abandonable(tt)
        kd = dom.kernel("decode/spin", _abi.BODY_SPIN, (600, 1, 1), _abi.SpinArgs(spin_out.data_ptr(), 10_000))
        kt = dom.kernel("train/gemm", _abi.BODY_GEMM_BF16, grid, a_co)
        dom.start()
        eng = Engine(dom, policy="tpot-first", lend_tenant=tt)
        jd = eng.add_job(td, _abi.LATENCY_CRITICAL)
        jt = eng.add_job(tt, _abi.BEST_EFFORT)
        eng.start()
        try:
            tr = [eng.submit(jt, [kt], "train/gemm", phase=_abi.TRAINING, grid_size=grid[0]) for _ in range(12)]
            import time
            dr = []
            for i in range(6):
                time.sleep(0.0015)
                dr.append(eng.submit(jd, [kd] * 3, "decode/spin", phase=_abi.DECODE, grid_size=600,
                                     saturation=Fraction(1, 2), tpot_ns=50_000_000))
            for r in dr + tr:
                eng.wait(r, 120000)
        finally:
            eng.stop()
            eng.close()
        blog = [b for b in dom.block_log() if b.tenant == tt]
        got = C_co.cpu()
    assert np.array_equal(got.view(torch.int16).numpy(), C_solo.cpu().view(torch.int16).numpy())
    seqs = sorted({b.seq for b in blog})
    assert len(seqs) == 12
    for s in seqs:
        assert sorted(b.block for b in blog if b.flags == 0 and b.seq == s) == list(range(grid[0]))
    print("abandoned attempts", sum(b.flags == 1 for b in blog))


def test_abandonable_tenant_mixed_bodies_no_deadlock():
    """an abandonable tenant whose program mixes bodies —
    a split-K abandonable GEMM, its split-K fold (not abandonable) and a plain
    GEMM — under 100% <-> 1/8 flips every 30 us.  Before the fix, lanes parked
    on launch s+1 (fold / plain GEMM waiting for s) while s's abandoned tiles
    sat in the retry ring with no lane left to run them.  Every launch must
    complete, bit-exact vs the same program run solo."""
    Ms, Ns, Ks, S = 2048, 2048, 4096, 4
    g = torch.Generator(device="cuda").manual_seed(11)
    A = ((torch.rand(Ms, Ks, device="cuda", generator=g) * 2 - 1)).to(torch.bfloat16)
    B = ((torch.rand(Ns, Ks, device="cuda", generator=g) * 2 - 1)).to(torch.bfloat16)
    ws = torch.zeros(_abi.splitk_ws_elems(Ms, Ns, 256, S), dtype=torch.float32, device="cuda")
    outs = {}
    for mode in ("solo", "co"):
        C1 = torch.zeros(Ms, Ns, dtype=torch.bfloat16, device="cuda")
        C2 = torch.zeros(Ms, Ns, dtype=torch.bfloat16, device="cuda")
        ab = 0 if mode == "solo" else 1
        a_split = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C1.data_ptr(), Ms, Ns, Ks, splits=S,
                                 ws=ws.data_ptr(), tma_store=False, abandon=ab)
        red_args, red_grid = _abi.splitk_reduce(ws.data_ptr(), C1.data_ptr(), Ms, Ns, Ks, 16, 256, S)
        a_plain = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C2.data_ptr(), Ms, Ns, Ks)
        gs, gp = _abi.gemm_grid(Ms, Ns, splits=S), _abi.gemm_grid(Ms, Ns)
        if mode == "solo":
            solo_launch(0, "split", _abi.BODY_GEMM_BF16, gs, a_split)
            solo_launch(0, "fold", _abi.BODY_SPLITK_REDUCE, red_grid, red_args)
            solo_launch(0, "plain", _abi.BODY_GEMM_BF16, gp, a_plain)
            torch.cuda.synchronize()
        else:
            with Domain(0, tiers=[Fraction(1)], block_log_capacity=0) as dom:
                t = dom.tenant("train", _abi.BEST_EFFORT)
                dom.set_abandonable(t)
                ks = dom.kernel("split", _abi.BODY_GEMM_BF16, gs, a_split)
                kr = dom.kernel("fold", _abi.BODY_SPLITK_REDUCE, red_grid, red_args)
                kp = dom.kernel("plain", _abi.BODY_GEMM_BF16, gp, a_plain)
                dom.start()
                n = dom.num_sms
                full, eighth = dom.mask(t, 0, n), dom.mask(t, 0, n // 8)
                dom.quota_set(full)
                dom.quota_periodic(30_000, full, eighth)
                last = None
                for _ in range(6):
                    dom.launch(t, ks)
                    dom.launch(t, kr)
                    last = dom.launch(t, kp)
                dom.wait(t, last, 120000)  # a deadlock times out here
                dom.quota_periodic(0, full, full)
        outs[mode] = (C1.cpu().view(torch.int16).numpy(), C2.cpu().view(torch.int16).numpy())
    assert np.array_equal(outs["solo"][0], outs["co"][0])
    assert np.array_equal(outs["solo"][1], outs["co"][1])
