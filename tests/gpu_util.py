"""Helpers for the -m gpu tests (device buffers via torch: plumbing only)."""
import ctypes

import torch


def dev_ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def sync():
    torch.cuda.synchronize()
