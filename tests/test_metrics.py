"""Metrics parity: ds_compute_metrics against the
reference's own compute_metrics (metrics.cpp:9-85, compiled into oracle/_ref)
on random request outcomes — TTFT/TPOT samples, nearest-rank p50/p90/p99
(exact), SLO violation counts, training kernel totals."""
import random
from fractions import Fraction

import pytest

from oracle import loader
from paper_2603_15042_b200.metrics import RequestOutcome, compute_metrics


def _random_outcomes(rnd, n):
    outs = []
    for _ in range(n):
        inference = rnd.random() < 0.8
        arrival = rnd.randint(0, 10**9)
        first = arrival + rnd.randint(0, 5 * 10**7)
        tokens = rnd.choice([0, 1, 2, 3, 8, 17, 128])
        last = first + rnd.randint(0, 10**8)
        slo = rnd.random() < 0.7
        outs.append(RequestOutcome(arrival=arrival, first_decode_finish=first, last_finish=last, output_tokens=tokens,
                                   inference=inference, completed=rnd.random() < 0.9,
                                   ttft_slo=rnd.randint(0, 5 * 10**7) if slo else None,
                                   tpot_slo=rnd.randint(0, 2 * 10**7) if slo else None,
                                   kernels_done=rnd.randint(0, 50)))
    return outs


@pytest.mark.parametrize("seed", range(6))
def test_compute_metrics_matches_reference(ref, seed):
    rnd = random.Random(seed)
    for n in (1, 2, 7, 100, 997):
        outs = _random_outcomes(rnd, n)
        makespan = rnd.randint(1, 10**10)
        got = compute_metrics(outs, makespan, kernels_completed=123)
        want = loader.ref_compute_metrics(
            [dict(inference=o.inference, completed=o.completed, output_tokens=o.output_tokens,
                  has_slo=o.ttft_slo is not None, arrival=o.arrival, first=o.first_decode_finish,
                  last=o.last_finish, ttft_slo=o.ttft_slo or 0, tpot_slo=o.tpot_slo or 0,
                  kernels_done=o.kernels_done) for o in outs], makespan, 123)
        for k in ("inference_completed", "training_kernels_completed", "tpot_excluded", "slo_requests",
                  "ttft_violations", "tpot_violations"):
            assert got[k] == want[k], k
        for k in ("inference_throughput", "training_throughput", "ttft_violation_rate", "tpot_violation_rate"):
            assert got[k] == pytest.approx(float(want[k]), rel=1e-12, abs=0), k
        for d in ("ttft", "tpot"):
            assert got[d]["count"] == want[f"{d}_count"]
            if got[d]["count"]:
                for p in ("p50", "p90", "p99"):
                    assert got[d][p] == want[f"{d}_{p}"], (d, p)      # exact
                assert got[d]["mean"] == pytest.approx(float(want[f"{d}_mean"]), rel=1e-12)


def test_nearest_rank_spec_example():
    # metrics.cpp:13: k = ceil(pct n / 100); 100 TPOT samples 1..100 -> p99 = 99, p50 = 50
    outs = [RequestOutcome(arrival=0, first_decode_finish=0, last_finish=i, output_tokens=2) for i in range(1, 101)]
    m = compute_metrics(outs, 1000)
    assert m["tpot"]["p99"] == 99 and m["tpot"]["p50"] == 50 and m["tpot"]["p90"] == 90
    # TPOT is exact: span 10 over 3 gaps
    m = compute_metrics([RequestOutcome(arrival=0, first_decode_finish=5, last_finish=15, output_tokens=4)], 20)
    assert m["tpot"]["p99"] == Fraction(10, 3) and m["ttft"]["p99"] == 5
