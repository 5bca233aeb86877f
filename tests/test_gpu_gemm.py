"""Training tenant: bf16 GEMM on tcgen05/TMEM.  Numerics vs a plain torch
fp32 reference (tolerance: bf16 output rounding, |err| <= 2^-7 |ref| + 2^-6),
and bit-exactness of the coroutine run (quota changes mid-kernel) vs solo."""
import numpy as np
import pytest
import torch

from paper_2603_15042_b200 import _abi
from paper_2603_15042_b200.runtime import Domain, solo_launch

pytestmark = pytest.mark.gpu


def make(M, N, K, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = (torch.rand(M, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    B = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    return A, B, C


@pytest.mark.parametrize("shape", [(128, 256, 64), (256, 512, 256), (512, 768, 1024), (384, 256, 4096)])
def test_gemm_solo_matches_fp32_reference(shape):
    M, N, K = shape
    A, B, C = make(M, N, K)
    args = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K)
    solo_launch(0, "gemm", _abi.BODY_GEMM_BF16, _abi.gemm_grid(M, N), args)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().t()
    err = (C.float() - ref).abs()
    tol = ref.abs() * 2 ** -7 + 2 ** -6
    assert bool((err <= tol).all()), float((err - tol).max())


def test_gemm_coroutine_bit_exact_vs_solo():
    M, N, K = 1024, 1024, 2048
    A, B, C_solo = make(M, N, K, seed=1)
    C_co = torch.zeros_like(C_solo)
    a_solo = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C_solo.data_ptr(), M, N, K)
    a_co = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C_co.data_ptr(), M, N, K)
    grid = _abi.gemm_grid(M, N)
    solo_launch(0, "gemm", _abi.BODY_GEMM_BF16, grid, a_solo)
    torch.cuda.synchronize()
    with Domain(0, block_log_capacity=1 << 16) as dom:
        dom.start()
        t = dom.tenant("train", _abi.BEST_EFFORT)
        dom.quota_set(dom.mask(t, 0, dom.num_sms))
        kid = dom.kernel("gemm", _abi.BODY_GEMM_BF16, grid, a_co, phase=_abi.TRAINING)
        nblk = grid[0]
        dom.quota_at_claim(t, 0, nblk // 3, dom.mask(t, 10, 20))
        dom.quota_at_claim(t, 0, 2 * nblk // 3, dom.mask(t, 0, dom.num_sms))
        s = dom.launch(t, kid)
        dom.wait(t, s)
        got = C_co.cpu()
        log = [b for b in dom.block_log() if b.tenant == t]
    assert sorted(b.block for b in log) == list(range(nblk))
    assert np.array_equal(got.view(torch.int16).numpy(), C_solo.cpu().view(torch.int16).numpy())


def run_split(A, B, C, M, N, K, bn, S, ws, dom=None, t=None, rows=16):
    args = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, bn=bn, splits=S,
                          ws=ws.data_ptr() if S > 1 else 0)
    grid = _abi.gemm_grid(M, N, bn, S)
    launches = [("gemm", _abi.BODY_GEMM_BF16, grid, args)]
    if S > 1:
        ra, rg = _abi.splitk_reduce(ws.data_ptr(), C.data_ptr(), M, N, K, 16, bn, S, rows)
        launches.append(("fold", _abi.BODY_SPLITK_REDUCE, rg, ra))
    if dom is None:
        for sid, body, g, a in launches:
            solo_launch(0, sid, body, g, a)
        torch.cuda.synchronize()
        return None
    kids = [dom.kernel(sid, body, g, a, phase=_abi.TRAINING) for sid, body, g, a in launches]
    seqs = [dom.launch(t, k) for k in kids]
    return seqs, grid[0]


@pytest.mark.parametrize("shape", [(256, 192, 128, 64, 1), (384, 384, 512, 128, 1), (128, 64, 4096, 64, 16),
                                   (256, 256, 2048, 128, 5), (128, 256, 3200, 256, 7)])
def test_gemm_tile_widths_and_splitk_match_fp32_reference(shape):
    """Config 4 GEMM variants: 128x64 / 128x128 tiles and split-K with the
    fixed-order fold launch."""
    M, N, K, bn, S = shape
    A, B, C = make(M, N, K, seed=3)
    ws = torch.zeros(max(1, _abi.splitk_ws_elems(M, N, bn, S)), device="cuda")
    run_split(A, B, C, M, N, K, bn, S, ws)
    ref = A.float() @ B.float().t()
    err = (C.float() - ref).abs()
    tol = ref.abs() * 2 ** -7 + 2 ** -6
    assert bool((err <= tol).all()), float((err - tol).max())


def test_splitk_coroutine_bit_exact_vs_solo():
    M, N, K, bn, S = 256, 192, 8192, 64, 12
    A, B, C_solo = make(M, N, K, seed=4)
    C_co = torch.zeros_like(C_solo)
    ws = torch.zeros(_abi.splitk_ws_elems(M, N, bn, S), device="cuda")
    run_split(A, B, C_solo, M, N, K, bn, S, ws)
    ws.zero_()
    with Domain(0, block_log_capacity=1 << 16) as dom:
        dom.start()
        t = dom.tenant("train", _abi.BEST_EFFORT)
        dom.quota_set(dom.mask(t, 0, 16))
        dom.quota_at_claim(t, 0, 20, dom.mask(t, 40, 60))
        seqs, nblk = run_split(A, B, C_co, M, N, K, bn, S, ws, dom, t)
        dom.wait(t, seqs[-1])
        got = C_co.cpu()
    assert np.array_equal(got.view(torch.int16).numpy(), C_solo.cpu().view(torch.int16).numpy())


@pytest.mark.parametrize("S", [5, 21])
def test_splitk_fold_row_groups_bit_identical(S):
    """The fold's row grouping (16 / 32 / 64 / 128 rows per block) is a launch
    shape only: every grouping gives the same bits, solo and as a coroutine;
    S = 21 covers the 8-partials-in-flight path and its remainder."""
    M, N, K, bn = 512, 256, 4096 if S == 5 else 21 * 512, 128
    A, B, C16 = make(M, N, K, seed=8)
    ws = torch.zeros(_abi.splitk_ws_elems(M, N, bn, S), device="cuda")
    run_split(A, B, C16, M, N, K, bn, S, ws, rows=16)
    for rows in (32, 64, 128):
        C = torch.zeros_like(C16)
        run_split(A, B, C, M, N, K, bn, S, ws, rows=rows)
        assert torch.equal(C.view(torch.int16), C16.view(torch.int16)), rows
    C_co = torch.zeros_like(C16)
    with Domain(0, block_log_capacity=0) as dom:
        dom.start()
        t = dom.tenant("train", _abi.BEST_EFFORT)
        dom.quota_set(dom.mask(t, 0, 24))
        seqs, _ = run_split(A, B, C_co, M, N, K, bn, S, ws, dom, t, rows=128)
        dom.wait(t, seqs[-1])
    assert torch.equal(C_co.view(torch.int16), C16.view(torch.int16))
    with pytest.raises(_abi.DsError):
        _abi.splitk_reduce(0, 0, M, N, K, 16, bn, S, rows=48)


@pytest.mark.parametrize("shape", [(128, 256, 64), (256, 512, 1024), (384, 768, 4096)])
def test_gemm_bk32_sw64_matches_fp32_reference(shape):
    """K blocks of 32 staged as SWIZZLE_64B tiles in a 4-stage ring."""
    M, N, K = shape
    A, B, C = make(M, N, K, seed=5)
    args = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, bk=32)
    solo_launch(0, "gemm", _abi.BODY_GEMM_BF16, _abi.gemm_grid(M, N), args)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().t()
    err = (C.float() - ref).abs()
    tol = ref.abs() * 2 ** -7 + 2 ** -6
    assert bool((err <= tol).all()), float((err - tol).max())


def test_gemm_bk32_coroutine_bit_exact_vs_solo():
    M, N, K = 1024, 1024, 2048
    A, B, C_solo = make(M, N, K, seed=6)
    C_co = torch.zeros_like(C_solo)
    grid = _abi.gemm_grid(M, N)
    solo_launch(0, "gemm", _abi.BODY_GEMM_BF16, grid, _abi.gemm_args(A.data_ptr(), B.data_ptr(), C_solo.data_ptr(), M, N, K, bk=32))
    torch.cuda.synchronize()
    a_co = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C_co.data_ptr(), M, N, K, bk=32)
    with Domain(0, block_log_capacity=0) as dom:
        dom.start()
        t = dom.tenant("train", _abi.BEST_EFFORT)
        dom.quota_set(dom.mask(t, 0, dom.num_sms))
        kid = dom.kernel("gemm", _abi.BODY_GEMM_BF16, grid, a_co, phase=_abi.TRAINING)
        dom.quota_at_claim(t, 0, grid[0] // 2, dom.mask(t, 0, 30))
        s = dom.launch(t, kid)
        dom.wait(t, s)
        got = C_co.cpu()
    assert np.array_equal(got.view(torch.int16).numpy(), C_solo.cpu().view(torch.int16).numpy())


def test_gemm_8192_coroutine_bit_exact_vs_solo_and_fp32():
    """The headline training tenant at full size: bf16 8192^3 (the config-2
    GEMM, group_m 32 as in the bench) as a coroutine under a device-timer quota
    flip 100% <-> 25% every 100 us (tiles revoked mid-kernel), bit-identical to
    the plain-grid solo launch; the solo result is within the bf16 tolerance of
    the fp32 product on a sample of 256 rows."""
    from paper_2603_15042_b200 import migration as mg
    M = N = K = 8192
    A, B, C_solo = make(M, N, K, seed=3)
    C_co = torch.zeros_like(C_solo)
    grid = _abi.gemm_grid(M, N)
    solo_launch(0, "gemm", _abi.BODY_GEMM_BF16, grid,
                _abi.gemm_args(A.data_ptr(), B.data_ptr(), C_solo.data_ptr(), M, N, K, group_m=32))
    torch.cuda.synchronize()
    rows = torch.arange(0, M, M // 256, device="cuda")
    ref = A[rows].float() @ B.float().t()
    err = (C_solo[rows].float() - ref).abs()
    assert bool((err <= ref.abs() * 2 ** -7 + 2 ** -5).all()), float((err - ref.abs() * 2 ** -7).max())
    a_co = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C_co.data_ptr(), M, N, K, group_m=32)
    with Domain(0, block_log_capacity=1 << 16) as dom:
        t = dom.tenant("train", _abi.BEST_EFFORT)
        kid = dom.kernel("gemm", _abi.BODY_GEMM_BF16, grid, a_co, phase=_abi.TRAINING)
        dom.start()
        r = mg.run(dom, t, kid, 100)
        blog = [b for b in dom.block_log() if b.tenant == t]
    assert r["flips"] >= 4
    assert sorted(b.block for b in blog if b.flags == 0) == list(range(grid[0]))
    assert torch.equal(C_co.view(torch.int16), C_solo.view(torch.int16))


@pytest.mark.parametrize("shape", [(12800, 256, 64, 128, 5), (25600, 64, 576, 64, 8), (3200, 128, 1152, 128, 3),
                                   (1280, 128, 192, 64, 7)])
def test_gemm_multi_tile_blocks_bit_exact_vs_one_tile(shape):
    """Multi-tile blocks (GemmArgs.tiles = T: T consecutive raster tiles per
    logical block, TMEM double-buffered, epilogue + TMA store overlapping the
    next tile's stream; ragged last block included) give C bit-identical to
    the one-tile records of the same tile width, solo and as a coroutine under
    mid-kernel quota changes, and within the bf16 tolerance of fp32."""
    M, N, K, bn, T = shape
    A, B, C_one = make(M, N, K, seed=5)
    C_multi, C_co = torch.zeros_like(C_one), torch.zeros_like(C_one)
    solo_launch(0, "gemm1", _abi.BODY_GEMM_BF16, _abi.gemm_grid(M, N, bn),
                _abi.gemm_args(A.data_ptr(), B.data_ptr(), C_one.data_ptr(), M, N, K, bn=bn))
    grid = _abi.gemm_grid(M, N, bn, tiles=T)
    assert grid[0] == -(-(M // 128) * (N // bn) // T)
    solo_launch(0, "gemmT", _abi.BODY_GEMM_BF16, grid,
                _abi.gemm_args(A.data_ptr(), B.data_ptr(), C_multi.data_ptr(), M, N, K, bn=bn, tiles=T))
    torch.cuda.synchronize()
    assert torch.equal(C_multi.view(torch.int16), C_one.view(torch.int16))
    rows = torch.arange(0, M, max(1, M // 256), device="cuda")
    ref = A[rows].float() @ B.float().t()
    err = (C_multi[rows].float() - ref).abs()
    assert bool((err <= ref.abs() * 2 ** -7 + 2 ** -6).all())
    a_co = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C_co.data_ptr(), M, N, K, bn=bn, tiles=T)
    with Domain(0, block_log_capacity=1 << 16) as dom:
        dom.start()
        t = dom.tenant("train", _abi.BEST_EFFORT)
        dom.quota_set(dom.mask(t, 0, dom.num_sms))
        kid = dom.kernel("gemmT", _abi.BODY_GEMM_BF16, grid, a_co, phase=_abi.TRAINING)
        nblk = grid[0]
        dom.quota_at_claim(t, 0, nblk // 3, dom.mask(t, 10, 20))
        dom.quota_at_claim(t, 0, 2 * nblk // 3, dom.mask(t, 0, dom.num_sms))
        s = dom.launch(t, kid)
        dom.wait(t, s)
        log = [b for b in dom.block_log() if b.tenant == t]
    assert sorted(b.block for b in log) == list(range(nblk))
    assert torch.equal(C_co.view(torch.int16), C_one.view(torch.int16))


def test_gemm_multi_tile_rejects_unsupported():
    from paper_2603_15042_b200._abi import DsError
    for kw in (dict(bn=256), dict(bn=128, splits=2, ws=1), dict(bn=128, abandon=True)):
        with pytest.raises(DsError):
            _abi.gemm_args(1, 1, 1, 1024, 1024, 1024, tiles=4, **kw)


@pytest.mark.parametrize("valid,bn,T", [((300, 200, 147), 64, 1), ((1000, 100, 100), 64, 2), ((147, 64, 5000), 64, 1)])
def test_gemm_valid_extents_read_no_padding(valid, bn, T):
    """Unpadded shapes inside tile-padded arrays (GemmArgs via valid=):
    the TMA loads zero-fill past (m, k) / (n, k), so garbage in the padding
    never reaches C, and the stores clip at (m, n), so C's padding keeps its
    contents (past n rounded up to 8: the 16-byte store unit writes zeros up
    to there); the valid block matches fp32 within the bf16 tolerance."""
    m, n, k = valid
    M, N, K = -(-m // 128) * 128, -(-n // bn) * bn, -(-k // 64) * 64
    A, B, _ = make(M, N, K, seed=9)
    A[m:, :] = float("nan")
    A[:, k:] = float("nan")
    B[n:, :] = float("nan")
    B[:, k:] = float("nan")
    C = torch.full((M, N), 7.0, device="cuda", dtype=torch.bfloat16)
    args = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, bn=bn, tiles=T, valid=(m, n, k))
    solo_launch(0, "gemm", _abi.BODY_GEMM_BF16, _abi.gemm_grid(M, N, bn, tiles=T), args)
    torch.cuda.synchronize()
    ref = A[:m, :k].float() @ B[:n, :k].float().t()
    got = C[:m, :n].float()
    assert bool(((got - ref).abs() <= ref.abs() * 2 ** -7 + 2 ** -6).all())
    n8 = -(-n // 8) * 8  # TMA stores clip at 16-byte granularity
    assert bool((C[m:, :] == 7.0).all()) and bool((C[:, n8:] == 7.0).all())
    assert bool((C[:m, n:n8] == 0.0).all())


@pytest.mark.parametrize("S", [2, 5, 8])
def test_splitk_fused_fold_bit_identical_to_fold_launch(S):
    """fuse_fold: the last-arriving split of each tile folds the S partials
    in split order inside the GEMM launch -- the same bits as the separate
    SPLITK_REDUCE launch, solo and as a coroutine under quota changes, and
    repeatable (the tickets come back to rest)."""
    M, N, K, bn = 512, 384, 64 * 8 * S, 128
    A, B, C_ref = make(M, N, K, seed=11)
    ws = torch.zeros(_abi.splitk_ws_elems(M, N, bn, S), device="cuda")
    run_split(A, B, C_ref, M, N, K, bn, S, ws, rows=64)
    wsf = torch.zeros(_abi.splitk_ws_elems(M, N, bn, S) + _abi.fold_tickets(M, N, bn), device="cuda")
    grid = _abi.gemm_grid(M, N, bn, S)
    for rep in range(2):
        C = torch.zeros_like(C_ref)
        args = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, bn=bn, splits=S, ws=wsf.data_ptr(),
                              fuse_fold=True)
        solo_launch(0, "gemm_ff", _abi.BODY_GEMM_BF16, grid, args)
        torch.cuda.synchronize()
        assert torch.equal(C.view(torch.int16), C_ref.view(torch.int16)), rep
    C_co = torch.zeros_like(C_ref)
    a_co = _abi.gemm_args(A.data_ptr(), B.data_ptr(), C_co.data_ptr(), M, N, K, bn=bn, splits=S, ws=wsf.data_ptr(),
                          fuse_fold=True)
    with Domain(0, block_log_capacity=0) as dom:
        dom.start()
        t = dom.tenant("train", _abi.BEST_EFFORT)
        dom.quota_set(dom.mask(t, 0, dom.num_sms))
        kid = dom.kernel("gemm_ff", _abi.BODY_GEMM_BF16, grid, a_co, phase=_abi.TRAINING)
        dom.quota_at_claim(t, 0, grid[0] // 3, dom.mask(t, 8, 30))
        dom.quota_at_claim(t, 0, 2 * grid[0] // 3, dom.mask(t, 0, dom.num_sms))
        for _ in range(3):
            s_last = dom.launch(t, kid)
        dom.wait(t, s_last)
    assert torch.equal(C_co.view(torch.int16), C_ref.view(torch.int16))
    assert int(wsf[-_abi.fold_tickets(M, N, bn):].view(torch.int32).abs().sum()) == 0
    with pytest.raises(_abi.DsError):
        _abi.gemm_args(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, bn=bn, fuse_fold=True)
