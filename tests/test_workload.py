"""Request streams + workload expansion (native, csrc/workload.cpp) against
the REFERENCE library compiled here (oracle/_ref) and the committed fixtures
(tests/golden/workload_golden.json, made by tests/golden/make_golden.py).
Bit-exact: arrival times as integers round(t*1e9), job round-robin, token
draws, expanded grids / decode indices / lab seeds."""
import json
import os
from fractions import Fraction

import pytest

from paper_2603_15042_b200 import workload as wl

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = [
    # (generator, rates, template kwargs, seed)
    ("burst", (1.0, 50.0, 2.0, 20.0, 100.0), dict(kind="inference", prompt_tokens=8, output_tokens=8), 0),
    ("burst", (1.0, 50.0, 2.0, 20.0, 100.0), dict(kind="inference", prompt_tokens=64, prompt_tokens_max=512,
                                                  output_tokens=4, output_tokens_max=64, streams=3), 4),
    ("burst", (0.0, 30.0, 0.5, 3.0, 17.5), dict(kind="inference", streams=2), 9),
    ("burst", (2.0, 0.0, 1.0, 4.0, 40.0), dict(kind="training", iterations=7, streams=2), 1),
    ("poisson", (3.0, 50.0), dict(kind="inference", prompt_tokens=1, prompt_tokens_max=9, output_tokens=2,
                                  output_tokens_max=3, streams=4), 7),
    ("poisson", (0.7, 300.0), dict(kind="training", iterations=0), 123456789),
    ("poisson", (0.0, 10.0), dict(), 1),  # empty stream
    ("burst", (1.0, 5.0, 3.0, 2.0, 10.0), dict(), 1),  # burst longer than the period: empty by definition
]


def native(gen, rates, tk, seed):
    t = wl.RequestTemplate(**tk)
    if gen == "poisson":
        return wl.gen_poisson(*rates, t, seed)
    return wl.gen_burst(*rates, t, seed)


def ref_records(gen, rates, tk, seed):
    from oracle import loader
    t = wl.RequestTemplate(**tk)
    text = loader.ref_gen_trace(gen, rates, 0 if t.kind == "inference" else 1, t.prompt_tokens, t.prompt_tokens_max,
                                t.output_tokens, t.output_tokens_max, t.iterations, t.streams, seed)
    return [json.loads(line) for line in text.splitlines() if line.strip()]


def as_tuple(r):
    return (r.arrival_q, r.job_id, r.kind, r.prompt_tokens if r.kind == "inference" else None,
            r.output_tokens if r.kind == "inference" else None, r.iterations if r.kind == "training" else None)


def ref_tuple(j):
    q = Fraction(j["arrival_time"]) * 10**9
    assert q.denominator == 1
    return (int(q), j["job_id"], j["kind"], j.get("prompt_tokens"), j.get("output_tokens"), j.get("iterations"))


@pytest.mark.parametrize("case", range(len(CASES)))
def test_generators_match_reference(ref, case):
    gen, rates, tk, seed = CASES[case]
    got = [as_tuple(r) for r in native(gen, rates, tk, seed)]
    want = [ref_tuple(j) for j in ref_records(gen, rates, tk, seed)]
    assert got == want


@pytest.mark.parametrize("case", range(len(CASES)))
def test_expand_matches_reference(ref, case):
    from oracle import loader
    gen, rates, tk, seed = CASES[case]
    reqs = native(gen, rates, tk, seed)
    text = "\n".join(json.dumps(j) for j in ref_records(gen, rates, tk, seed))
    want = []
    for line in loader.ref_expand(text, 8, 164, 2048, 5).splitlines():
        job, phase, grid, di, req, sd, arr = line.split()
        want.append((int(job), int(phase), int(grid), int(di), int(req), int(sd), int(Fraction(arr) * 10**9)))
    got = [(k.job, k.phase, k.grid_size, k.decode_index, k.request, k.lab_seed, k.arrival_q)
           for k in wl.expand_workload(reqs, 8, 164, 2048, 5)]
    assert got == want


def test_generators_match_golden():
    g = json.load(open(os.path.join(HERE, "golden", "workload_golden.json")))
    for c in g["cases"]:
        got = [list(as_tuple(r)) for r in native(c["gen"], tuple(c["rates"]), c["template"], c["seed"])]
        assert got == c["records"], c["gen"]
        plan = [[k.job, k.phase, k.grid_size, k.decode_index, k.request, k.lab_seed]
                for k in wl.expand_workload(native(c["gen"], tuple(c["rates"]), c["template"], c["seed"]), 8, 164,
                                            2048, 5)]
        assert plan == c["plan"]


def test_spec_burst_shape():
    """gen_burst(base=1, burst=50, burst_dur=2, period=20): arrivals cluster in
    the first 2 units of each period."""
    reqs = native(*CASES[0][:3], 0)
    inb = sum(1 for r in reqs if (r.arrival_q % (20 * 10**9)) < 2 * 10**9)
    assert len(reqs) > 0 and inb / len(reqs) > 0.8
    assert all(b.arrival_q >= a.arrival_q for a, b in zip(reqs, reqs[1:]))


def test_invalid_template_raises():
    with pytest.raises(Exception):
        wl.gen_poisson(1.0, 1.0, wl.RequestTemplate(kind="bogus"), 0)


def test_mixed_job_kinds_rejected():
    a = wl.Request(0, "job-0", 0, "inference", 8, 2, 0)
    b = wl.Request(1, "job-0", 0, "training", 0, 0, 3)
    with pytest.raises(Exception):
        wl.expand_workload([a, b])
