"""Workload-aware placement of a tenant mix across GPUs (config 5) and the
per-rank view of it.  The decision is native (csrc/placement.cpp,
``ds_place_tenants``); every rank computes the same map from the same
seeded tenant list, so no collective is needed to agree on it.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Sequence

from . import _abi
from ._abi import check, lib


@dataclass
class TenantSpec:
    name: str
    kind: str              # "decode" | "train"
    priority: int          # _abi.LATENCY_CRITICAL | _abi.BEST_EFFORT
    hbm_frac: float
    tensor_frac: float
    mem_gb: float
    size: int = 0          # decode: layers; train: GEMM edge


def place(tenants: Sequence[TenantSpec], n_devices: int, mem_cap_gb: float = 0.0) -> List[int]:
    n = len(tenants)
    arr = (_abi.TenantDemand * max(1, n))()
    for i, t in enumerate(tenants):
        arr[i] = _abi.TenantDemand(t.priority, _abi.DECODE if t.kind == "decode" else _abi.TRAINING, t.hbm_frac,
                                   t.tensor_frac, t.mem_gb)
    out = (ctypes.c_int32 * max(1, n))()
    check(lib().ds_place_tenants(arr, n, n_devices, mem_cap_gb, out))
    return list(out[:n])


def config5_mix(n: int = 16) -> List[TenantSpec]:
    """The synthetic 16-tenant mix of config 5: 8 decode tenants
    (Llama-3-8B-shaped layers, batch 32, KV 1024; 2..8 layers) and 8 training
    tenants (bf16 GEMMs, 2048^3 .. 8192^3).  Demands are the roofline shares
    of one B200 (decode: weight+KV bytes at HBM peak over a 10 ms TPOT budget;
    training: fraction of tensor peak a tenant can keep busy)."""
    out = []
    layer_bytes = 436.2e6 + 4.19e6 * 32  # weights + KV per layer (batch 32, L = 1024)
    for i in range(n // 2):
        layers = (2, 4, 6, 8)[i % 4]
        hbm = layers * layer_bytes / 6553.6e9 / 10e-3
        out.append(TenantSpec(f"decode{i}", "decode", _abi.LATENCY_CRITICAL, round(hbm, 4), 0.02,
                              round(2.2 * layers * layer_bytes / 1e9 + 2.1, 2), layers))
    for i in range(n // 2):
        edge = (2048, 4096, 6144, 8192)[i % 4]
        out.append(TenantSpec(f"train{i}", "train", _abi.BEST_EFFORT, 0.05, round(min(1.0, (edge / 8192) ** 1.5), 4),
                              round(3 * edge * edge * 2 / 1e9, 3), edge))
    return out
