"""Helpers for the -m gpu tests (device buffers via torch: plumbing only)."""
import ctypes

import torch


def dev_ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def sync():
    torch.cuda.synchronize()


def sgemm_copies(M=1024, N=1024, K=1024, copies=1):
    """fp32 SGEMM inputs and copies+1 outputs; the solo result is in Cs[0]."""
    from paper_2603_15042_b200 import _abi
    from paper_2603_15042_b200.runtime import solo_launch
    g = torch.Generator(device="cuda").manual_seed(11)
    A = torch.rand(M, K, device="cuda", generator=g) * 2 - 1
    B = torch.rand(K, N, device="cuda", generator=g) * 2 - 1
    Cs = [torch.zeros(M, N, device="cuda") for _ in range(copies + 1)]
    args = [_abi.SgemmArgs(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, 0) for C in Cs]
    grid = (N // 64, M // 64, 1)
    solo_launch(0, "sgemm", _abi.BODY_SGEMM, grid, args[0])  # reference result in Cs[0]
    torch.cuda.synchronize()
    return (A, B, Cs), args, grid
