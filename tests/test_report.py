"""Report schema parity: metrics_to_json and run_compare output carry exactly
the reference's keys, nesting and order (metrics.cpp:132-166,
corosim.cpp:99-123), checked against the compiled reference's own report of a
scenario; values agree where both compute the same quantity (counts)."""
import json
from fractions import Fraction

from paper_2603_15042_b200 import metrics as M
from paper_2603_15042_b200 import report


def _keys(d):
    return [(k, _keys(v) if isinstance(v, dict) else None) for k, v in d.items()]


def _scenario():
    recs = [{"arrival_time": "0", "job_id": "train", "kind": "training", "iterations": 6, "priority": "best_effort"}]
    recs += [{"arrival_time": str(i), "job_id": "chat", "kind": "inference", "prompt_tokens": 16,
              "output_tokens": 4, "priority": "latency_critical"} for i in range(5)]
    return {"devices": [{"tiers": ["0.25", "0.5", "1"]}], "policy": "tpot-first",
            "slo": {"ttft": "4", "tpot": "2"}, "workload": {"records": recs}}


def test_metrics_json_schema_matches_reference(ref):
    from oracle import loader
    r = json.loads(loader.ref_simulate(json.dumps(_scenario())))
    ref_m = r["metrics"]
    outs = [M.RequestOutcome(arrival=i * 1000, first_decode_finish=i * 1000 + 500, last_finish=i * 1000 + 900,
                             output_tokens=4, ttft_slo=4000, tpot_slo=2000, kernels_done=5) for i in range(5)]
    m = M.compute_metrics(outs, makespan_ns=10_000, kernels_completed=31)
    ledger = {"ctx_switches": 2, "ctx_switch_total_ns": 10, "preemptions": 1, "preempt_total_ns": 5,
              "migrations": 3, "migration_total_ns": 7, "demand_faults": 0, "demand_fault_total_ns": 0}
    mine = report.metrics_to_json(m, ledger)
    ref_core = {k: v for k, v in ref_m.items() if k not in ("normalized_throughput", "aggregate_normalized")}
    assert _keys(mine) == _keys(ref_core)
    assert mine["overheads"]["total_added_latency"] == "22"
    # the counts the reference reports for its own run have the same meaning here
    assert ref_m["inference_completed"] == 5 and mine["inference_completed"] == 5
    norm = report.metrics_to_json(m, ledger, {0: Fraction(1, 2), 1: Fraction(1)})
    assert list(norm)[-2:] == ["normalized_throughput", "aggregate_normalized"]
    assert norm["aggregate_normalized"] == "1.5"


def test_compare_pairs_two_runs_like_run_compare():
    outs = [M.RequestOutcome(arrival=0, first_decode_finish=10, last_finish=40, output_tokens=4)]
    a = report.metrics_to_json(M.compute_metrics(outs, 100, 4))
    b = report.metrics_to_json(M.compute_metrics(outs, 200, 4))
    c = report.compare(a, b, "config2", "tpot-first", "config2", "temporal")
    assert list(c) == ["a", "b"]
    assert c["a"]["policy"] == "tpot-first" and c["b"]["policy"] == "temporal"
    assert list(c["a"])[-2:] == ["scenario", "policy"]
