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
