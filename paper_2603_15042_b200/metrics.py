"""Request metrics over measured outcomes: ds_compute_metrics, the
reference's compute_metrics (proj/src/io/metrics.cpp:9-85) on integer-ns
device timestamps (TTFT to the first decode finish, TPOT over tokens - 1,
nearest-rank percentiles, SLO violations)."""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from fractions import Fraction
from typing import Sequence

from . import _abi
from ._abi import check, lib


@dataclass
class RequestOutcome:
    """RequestOutcome + RequestMeta (engine.hpp:50-57,117-125), times in ns."""
    arrival: int
    first_decode_finish: int
    last_finish: int
    output_tokens: int
    inference: bool = True
    completed: bool = True
    ttft_slo: int | None = None
    tpot_slo: int | None = None
    kernels_done: int = 0


def compute_metrics(outcomes: Sequence[RequestOutcome], makespan_ns: int, kernels_completed: int = 0) -> dict:
    n = len(outcomes)
    arr = (_abi.RequestOutcome * max(1, n))()
    for i, o in enumerate(outcomes):
        has_slo = o.ttft_slo is not None or o.tpot_slo is not None
        arr[i] = _abi.RequestOutcome(int(o.inference), int(o.completed), o.output_tokens, int(has_slo), o.arrival,
                                     o.first_decode_finish, o.last_finish, o.ttft_slo or 0, o.tpot_slo or 0,
                                     o.kernels_done)
    m = _abi.Metrics()
    check(lib().ds_compute_metrics(arr, n, makespan_ns, kernels_completed, ctypes.byref(m)))

    def dist(d):
        out = {"count": d.count}
        if d.count:
            out.update(mean=d.mean, p50=Fraction(d.p50_num, d.p50_den), p90=Fraction(d.p90_num, d.p90_den),
                       p99=Fraction(d.p99_num, d.p99_den))
        return out

    return {"makespan_ns": m.makespan_ns, "kernels_completed": m.kernels_completed,
            "inference_completed": m.inference_completed,
            "training_kernels_completed": m.training_kernels_completed,
            "inference_throughput": m.inference_throughput, "training_throughput": m.training_throughput,
            "ttft": dist(m.ttft), "tpot": dist(m.tpot), "tpot_excluded": m.tpot_excluded,
            "slo_requests": m.slo_requests, "ttft_violations": m.ttft_violations,
            "tpot_violations": m.tpot_violations, "ttft_violation_rate": m.ttft_violation_rate,
            "tpot_violation_rate": m.tpot_violation_rate}
