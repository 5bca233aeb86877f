"""Integer-bookkeeping parity with the reference simulator (SURVEY §8a rows
a1/a18, §7 step 4): on the same two-job trace (training iterations + bursty
inference requests from gen_burst), the GPU engine's per-vctx transcripts
(executed (semantic_id, grid_size) in completion order), logical progress
and completed-kernel count equal the reference SimEngine's
(tests/golden/transcript_golden.json, made by tests/golden/make_golden.py
from oracle/_ref).  The kernels themselves are test bodies (spin) — the
bookkeeping, not the arithmetic, is under test here."""
import json
import os
from fractions import Fraction

import pytest

from paper_2603_15042_b200 import workload as wl

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "transcript_golden.json")
TRAIN_ITERS = 12


def trace():
    return wl.gen_burst(1.0, 6.0, 2.0, 10.0, 20.0, wl.RequestTemplate(prompt_tokens=8, prompt_tokens_max=40,
                                                                      output_tokens=2, output_tokens_max=5), seed=3)


def decimal(q: int) -> str:
    return f"{q // 10**9}.{q % 10**9:09d}"


def scenario():
    reqs = trace()
    recs = [{"arrival_time": "0", "job_id": "train", "kind": "training", "iterations": TRAIN_ITERS,
             "priority": "best_effort"}]
    recs += [{"arrival_time": decimal(r.arrival_q), "job_id": "chat", "kind": "inference",
              "prompt_tokens": r.prompt_tokens, "output_tokens": r.output_tokens, "priority": "latency_critical"}
             for r in reqs]
    return {"devices": [{"tiers": ["0.25", "0.5", "1"]}], "policy": "tpot-first", "workload": {"records": recs}}, reqs


def log_projection(lines):
    """Event log (reference schema, engine.cpp:316-329) -> per-vctx streams of
    first starts and finishes [kind, kernel, grid] (timing-independent: the
    transcript order), and the field names each logged kind carries."""
    streams, schema = {}, {}
    for line in lines:
        e = json.loads(line) if isinstance(line, str) else line
        k = e["kind"]
        if k in ("KernelStart", "KernelFinish") and "kernel" in e:
            schema.setdefault(k, sorted(e.keys()))
            if k == "KernelFinish" or not e.get("resumed"):
                streams.setdefault(str(e["vctx"]), []).append([k, e["kernel"], e["grid"]])
    return streams, schema


def expected_plan():
    """(job, semantic_id, grid) per kernel in expansion order: job 0 = train, 1 = chat."""
    _, reqs = scenario()
    train = wl.Request(0, "train-0", 0, "training", 0, 0, TRAIN_ITERS)
    chat = [wl.Request(r.arrival_q, "chat-0", 1, "inference", r.prompt_tokens, r.output_tokens, 0) for r in reqs]
    names = {0: "prefill/default", 1: "decode/default", 2: "train/default"}
    return [(k.job, names[k.phase], k.grid_size) for k in wl.expand_workload([train] + chat, 8, 8, 128, 50)]


def test_reference_transcripts_are_the_expansion_order():
    g = json.load(open(GOLD))
    plan = expected_plan()
    for job in (0, 1):
        assert [list(x[1:]) for x in plan if x[0] == job] == g["transcripts"][str(job)]
        assert g["logical_progress"][str(job)] == sum(1 for x in plan if x[0] == job)
    assert g["kernels_completed"] == len(plan)


@pytest.mark.gpu
def test_gpu_engine_transcripts_match_reference():
    import torch
    from paper_2603_15042_b200 import _abi
    from paper_2603_15042_b200.runtime import Domain, Engine
    g = json.load(open(GOLD))
    plan = expected_plan()
    out = torch.empty(3 * 256, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    tiers = [Fraction(1, 4), Fraction(1, 2), Fraction(1)]
    phase = {"prefill/default": _abi.PREFILL, "decode/default": _abi.DECODE, "train/default": _abi.TRAINING}
    with Domain(0, tiers=tiers, block_log_capacity=0) as dom:
        tenants = [dom.tenant("train", _abi.BEST_EFFORT), dom.tenant("chat", _abi.LATENCY_CRITICAL)]
        kid = {}
        for _, sid, grid in plan:
            if (sid, grid) not in kid:
                kid[(sid, grid)] = dom.kernel(sid, _abi.BODY_SPIN, (grid, 1, 1), _abi.SpinArgs(out.data_ptr(), 2000))
        dom.start()
        eng = Engine(dom, policy="tpot-first", lend_tenant=tenants[0], capture_log=True)
        jobs = [eng.add_job(tenants[0], _abi.BEST_EFFORT), eng.add_job(tenants[1], _abi.LATENCY_CRITICAL)]
        eng.start()
        try:
            sig = {}
            last = []
            for job, sid, grid in plan:
                r = eng.submit(jobs[job], [kid[(sid, grid)]], sid, phase[sid], grid_size=grid, base_hint_ns=100_000,
                               saturation=Fraction(1, 2))
                sig[r] = [sid, grid]
                last.append(r)
            for r in last:
                eng.wait(r, 60000)
            got = {str(j): [sig[r] for r in eng.transcript(jobs[j])] for j in (0, 1)}
            completed = eng.counters()["completed"]
            log = eng.event_log()
        finally:
            eng.stop()
            eng.close()
    assert got == g["transcripts"]
    assert {j: len(v) for j, v in got.items()} == g["logical_progress"]
    assert completed == g["kernels_completed"]
    # event log: the reference's schema for every start / finish line, and the
    # same per-vctx first-start / finish streams as the reference's own log
    streams, schema = log_projection(log)
    assert schema == g["log_schema"]
    assert streams == g["log_streams"]
