"""Reports in the reference's schema: metrics_to_json (proj/src/io/metrics.cpp:
132-166) over measured device-ns metrics, and run_compare's paired output
(tools/corosim.cpp:99-123): {"a": metrics + scenario + policy, "b": ...}.

Times are integer ns (the reference prints its model units); every key, its
nesting and order follow the reference so a reader of corosim's reports reads
these unchanged."""
from __future__ import annotations

from fractions import Fraction
from typing import Dict, Optional


def _dec(x) -> str:
    """to_decimal_string for the exact values the native metrics return
    (Fraction percentiles, integer ns), plain repr for doubles."""
    if isinstance(x, Fraction):
        if x.denominator == 1:
            return str(x.numerator)
        return f"{float(x):.12f}".rstrip("0").rstrip(".")
    if isinstance(x, float):
        return f"{x:.12f}".rstrip("0").rstrip(".") if x != int(x) else str(int(x))
    return str(x)


def _dist(d: dict) -> dict:
    out = {"count": d["count"]}
    if d["count"]:
        for k in ("mean", "p50", "p90", "p99"):
            out[k] = _dec(d[k])
    return out


def metrics_to_json(m: dict, ledger: Optional[dict] = None, normalized: Optional[Dict[int, Fraction]] = None) -> dict:
    """m: metrics.compute_metrics(...) output; ledger: the OverheadLedger
    fields (ns totals, counts) as ds_ledger_get / bench 'ledger' report them;
    normalized: job -> solo span / shared span (add_normalization)."""
    L = ledger or {}
    tot = sum(L.get(k, 0) for k in ("ctx_switch_total_ns", "preempt_total_ns", "migration_total_ns",
                                     "demand_fault_total_ns"))
    j = {
        "makespan": _dec(m["makespan_ns"]),
        "kernels_completed": m["kernels_completed"],
        "inference_completed": m["inference_completed"],
        "training_kernels_completed": m["training_kernels_completed"],
        "inference_throughput": _dec(float(m["inference_throughput"])),
        "training_throughput": _dec(float(m["training_throughput"])),
        "ttft": _dist(m["ttft"]),
        "tpot": _dist(m["tpot"]),
        "tpot_excluded": m["tpot_excluded"],
        "slo": {"requests": m["slo_requests"], "ttft_violations": m["ttft_violations"],
                "tpot_violations": m["tpot_violations"],
                "ttft_violation_rate": _dec(float(m["ttft_violation_rate"])),
                "tpot_violation_rate": _dec(float(m["tpot_violation_rate"]))},
        "overheads": {"ctx_switch_total": _dec(L.get("ctx_switch_total_ns", 0)),
                      "ctx_switches": L.get("ctx_switches", 0),
                      "preempt_total": _dec(L.get("preempt_total_ns", 0)),
                      "preemptions": L.get("preemptions", 0),
                      "migration_total": _dec(L.get("migration_total_ns", 0)),
                      "migrations": L.get("migrations", 0),
                      "demand_fault_total": _dec(L.get("demand_fault_total_ns", 0)),
                      "demand_faults": L.get("demand_faults", 0),
                      "total_added_latency": _dec(tot)},
    }
    if normalized:
        j["normalized_throughput"] = {str(k): _dec(Fraction(v)) for k, v in sorted(normalized.items())}
        j["aggregate_normalized"] = _dec(sum(Fraction(v) for v in normalized.values()))
    return j


def compare(a: dict, b: dict, scenario_a: str, policy_a: str, scenario_b: str, policy_b: str) -> dict:
    """run_compare (corosim.cpp:99-123): the two runs' metrics side by side."""
    out = {"a": dict(a), "b": dict(b)}
    out["a"]["scenario"], out["a"]["policy"] = scenario_a, policy_a
    out["b"]["scenario"], out["b"]["policy"] = scenario_b, policy_b
    return out
