"""Cross-check the restatements against the REFERENCE library compiled here
(oracle/_ref, built from /root/reference/proj/src with the GMP Boost shim)."""
import json
import random
from fractions import Fraction as F

import pytest

from oracle import loader, numlab as nl


@pytest.mark.parametrize("fmt", [nl.FP16, nl.BF16, nl.FP32])
def test_reduction_result_matches_reference(ref, cn, fmt):
    code = loader.FMT_CODE[fmt]
    for seed in range(4):
        for g in (1, 2, 7, 64, 4096, 5000):
            r = loader.ref_reduction_result(seed, 4096, fmt, g)
            assert nl.encode_bits(fmt, r) == cn.cn_reduction_result(seed, 4096, code, g)


def test_round_to_matches_reference(ref):
    rnd = random.Random(99)
    for _ in range(300):
        fmt = rnd.choice([nl.FP16, nl.BF16, nl.FP32])
        x = F(rnd.randint(-2**40, 2**40), 2**rnd.randint(0, 170))
        assert loader.ref_round_to(fmt, x) == nl.round_to(fmt, x)


def test_reduce_values_tree_matches_reference(ref):
    rnd = random.Random(3)
    for fmt in (nl.FP16, nl.BF16, nl.FP32):
        vals = [nl.round_to(fmt, F(rnd.randint(-2**16, 2**16), 2**12)) for _ in range(37)]
        for g in (1, 3, 8, 37):
            for tree in (False, True):
                want = loader.ref_reduce_values(fmt, vals, g, tree)
                assert nl.reduce_with_plan(vals, fmt, nl.balanced_bounds(37, g), tree) == want


def test_reference_simulator_runs(ref):
    sc = {"devices": [{"tiers": ["0.25", "0.5", "1"]}], "policy": "tpot-first",
          "workload": {"records": [
              {"arrival_time": "0", "job_id": "train", "kind": "training", "iterations": 4,
               "priority": "best_effort"},
              {"arrival_time": "1", "job_id": "chat", "kind": "inference", "prompt_tokens": 64,
               "output_tokens": 4, "priority": "latency_critical",
               "slo": {"ttft": "2", "tpot": "0.5"}}]}}
    out = json.loads(loader.ref_simulate(json.dumps(sc)))
    assert out["kernels_completed"] == 4 + 1 + 4
    eq = json.loads(loader.ref_equivalence(json.dumps(sc)))
    assert eq["equivalent"] is True


def _bench_scenario(dbw, tbw):
    recs = [{"arrival_time": "0", "job_id": "train", "kind": "training", "iterations": 352,
             "priority": "best_effort", "profile": "gemm"}]
    for r in range(3):
        recs.append({"arrival_time": str(29000 + r * 116000), "job_id": "chat", "kind": "inference",
                     "prompt_tokens": 8, "output_tokens": 8, "priority": "latency_critical",
                     "slo": {"ttft": "21900", "tpot": "10950"}})
    return {"devices": [{"tiers": ["0.25", "0.5", "0.75", "1"]}], "policy": "tpot-first",
            "policy_params": {"quantum": "5000"}, "segments_per_kernel": 16, "event_budget": 100000000,
            "profiles": {"inference": {"default": {"decode_cost": "7300", "prefill_cost_per_token": "1",
                                                   "decode_saturation": "0.75", "decode_mem_bound": "0.8",
                                                   "decode_bw_demand": dbw, "decode_grid": 164}},
                         "training": {"gemm": {"iteration_cost": "1000", "saturation": "0.25",
                                               "mem_bound": "0.1", "bw_demand": tbw, "grid": 2048}}},
            "workload": {"records": recs}}


def test_reference_assertion_is_reported_not_fatal(ref):
    # bench.py's scenario runs with bandwidth demands summing to 1 ...
    out = json.loads(loader.ref_simulate(json.dumps(_bench_scenario("0.75", "0.25"))))
    assert out["metrics"]["tpot"]["p99"] is not None
    # ... and an oversubscribed HBM trips the reference's own work-conservation
    # assert (engine.cpp:838); the harness turns it into an error, not an abort
    with pytest.raises(RuntimeError, match="work_done"):
        loader.ref_simulate(json.dumps(_bench_scenario("0.9", "0.2")))
    # the library is still usable afterwards
    out = json.loads(loader.ref_simulate(json.dumps(_bench_scenario("0.75", "0.25"))))
    assert out["metrics"]["tpot"]["p99"] is not None
