"""Request streams and workload expansion over the native library.

Mirrors the reference's generator API (proj/include/corosim/io/trace.hpp:41-65:
``RequestTemplate``, ``gen_poisson``, ``gen_burst``) and ``expand_workload``
(proj/include/corosim/io/workload.hpp:61-62).  The arithmetic runs in
libdetshare.so (csrc/workload.cpp); arrivals come back as exact integers
``arrival_q = round(t * 1e9)`` in the trace's time unit, the numerator of
the reference's quantised Rational over 10^9.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List

from . import _abi
from ._abi import check, lib


@dataclass
class RequestTemplate:
    kind: str = "inference"  # "inference" | "training"
    prompt_tokens: int = 256
    prompt_tokens_max: int = 0
    output_tokens: int = 32
    output_tokens_max: int = 0
    iterations: int = 50
    streams: int = 1
    job_prefix: str = "job"

    def c(self) -> _abi.RequestTemplate:
        if self.kind not in ("inference", "training"):
            raise _abi.DsError(105, f"unknown request kind {self.kind!r}")
        return _abi.RequestTemplate(_abi.REQ_INFERENCE if self.kind == "inference" else _abi.REQ_TRAINING,
                                    self.prompt_tokens, self.prompt_tokens_max, self.output_tokens,
                                    self.output_tokens_max, self.iterations, self.streams)


@dataclass
class Request:
    arrival_q: int       # round(arrival * 1e9)
    job_id: str
    stream: int
    kind: str
    prompt_tokens: int
    output_tokens: int
    iterations: int

    @property
    def arrival(self) -> float:
        return self.arrival_q / 1e9


def _collect(fn, tmpl: RequestTemplate, *args) -> List[Request]:
    ct = tmpl.c()
    n = ctypes.c_int64()
    check(fn(*args[:-1], ctypes.byref(ct), args[-1], None, 0, ctypes.byref(n)))
    buf = (_abi.Request * max(1, n.value))()
    check(fn(*args[:-1], ctypes.byref(ct), args[-1], buf, n.value, ctypes.byref(n)))
    return [Request(r.arrival_q, f"{tmpl.job_prefix}-{r.stream}", r.stream,
                    "inference" if r.kind == _abi.REQ_INFERENCE else "training", r.prompt_tokens,
                    r.output_tokens, r.iterations) for r in buf[:n.value]]


def gen_poisson(rate: float, duration: float, tmpl: RequestTemplate, seed: int) -> List[Request]:
    """Poisson arrivals at `rate` over [0, duration) (trace.cpp:189-202)."""
    return _collect(lib().ds_gen_poisson, tmpl, float(rate), float(duration), seed)


def gen_burst(base_rate: float, burst_rate: float, burst_duration: float, period: float, duration: float,
              tmpl: RequestTemplate, seed: int) -> List[Request]:
    """Rate alternates base/burst; each period opens with `burst_duration`
    at the burst rate (trace.cpp:204-232)."""
    return _collect(lib().ds_gen_burst, tmpl, float(base_rate), float(burst_rate), float(burst_duration),
                    float(period), float(duration), seed)


@dataclass
class KernelPlan:
    request: int
    job: int
    phase: int
    decode_index: int
    grid_size: int
    arrival_q: int
    lab_seed: int


def expand_workload(reqs: List[Request], tokens_per_grid_unit: int = 8, decode_grid: int = 8,
                    train_grid: int = 128, default_iterations: int = 50) -> List[KernelPlan]:
    """Request -> kernel records (workload.cpp:51-174), in request order."""
    arr = (_abi.Request * max(1, len(reqs)))()
    for i, r in enumerate(reqs):
        arr[i] = _abi.Request(r.arrival_q, r.stream, _abi.REQ_INFERENCE if r.kind == "inference" else _abi.REQ_TRAINING,
                              r.prompt_tokens, r.output_tokens, r.iterations, 0)
    p = _abi.ExpandParams(tokens_per_grid_unit, decode_grid, train_grid, default_iterations, 0)
    n = ctypes.c_int64()
    check(lib().ds_expand_workload(arr, len(reqs), ctypes.byref(p), None, 0, ctypes.byref(n)))
    out = (_abi.KernelPlan * max(1, n.value))()
    check(lib().ds_expand_workload(arr, len(reqs), ctypes.byref(p), out, n.value, ctypes.byref(n)))
    return [KernelPlan(k.request, k.job, k.phase, k.decode_index, k.grid_size, k.arrival_q, k.lab_seed)
            for k in out[:n.value]]
