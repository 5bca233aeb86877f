"""Generate tests/golden/*.json from the REFERENCE library compiled here
(oracle/_ref/libcorosim_ref.so built from /root/reference by oracle/Makefile).

Committed with its outputs: the GPU box has no /root/reference, so GPU parity
tests read these fixtures instead of calling the reference.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from oracle import loader, numlab as nl  # noqa: E402


def main():
    assert loader.reference() is not None, "needs /root/reference (reference build)"
    out = {"source": "oracle/_ref (reference corosim compiled from /root/reference)",
           "n": 4096, "cases": []}
    for fmt in (nl.FP16, nl.BF16, nl.FP32):
        for seed in range(8):
            for g in (1, 2, 3, 7, 16, 37, 64, 148):
                fv = loader.ref_reduction_result(seed, 4096, fmt, g)
                out["cases"].append({"fmt": fmt, "seed": seed, "grid": g,
                                     "bits": nl.encode_bits(fmt, fv)})
    # ragged / edge: n < g (empty chunks), n = 1, n = 0
    for fmt in (nl.FP16, nl.BF16, nl.FP32):
        for (n, g) in ((5, 8), (1, 1), (1, 4), (0, 3), (13, 13), (100, 99)):
            fv = loader.ref_reduction_result(11, n, fmt, g)
            out["cases"].append({"fmt": fmt, "seed": 11, "grid": g, "n": n,
                                 "bits": nl.encode_bits(fmt, fv)})
    with open(os.path.join(HERE, "reduction_golden.json"), "w") as f:
        json.dump(out, f, indent=0)
    # SPEC.md:391-393 round_to examples + a few derived edge values via the reference
    from fractions import Fraction as F
    rt = []
    for fmt, x in ((nl.FP16, F(1)), (nl.FP16, 1 + F(1, 2**11)), (nl.BF16, 1 + F(1, 2**8)),
                   (nl.FP16, F(65520)), (nl.FP16, F(65519)), (nl.FP16, F(1, 2**25)),
                   (nl.FP16, F(3, 2**26)), (nl.FP16, -F(1, 2**26)), (nl.BF16, F(1, 3)),
                   (nl.FP32, F(1, 3)), (nl.FP32, F(2**128)), (nl.FP32, F(1, 2**150)),
                   (nl.FP32, F(3, 2**150)), (nl.BF16, -F(7, 5))):
        fv = loader.ref_round_to(fmt, x)
        rt.append({"fmt": fmt, "num": x.numerator, "den": x.denominator, "cls": fv.cls,
                   "bits": nl.encode_bits(fmt, fv)})
    with open(os.path.join(HERE, "round_to_golden.json"), "w") as f:
        json.dump({"source": out["source"], "cases": rt}, f, indent=0)
    print("wrote", len(out["cases"]), "reduction cases,", len(rt), "round_to cases")
    # request streams + expansion (trace.cpp:189-232, workload.cpp:51-174) from the reference
    import test_workload as tw  # noqa: E402  (tests/ on sys.path below)
    wcases = []
    for gen, rates, tk, seed in tw.CASES[:4]:
        recs = [list(tw.ref_tuple(j)) for j in tw.ref_records(gen, rates, tk, seed)]
        text = "\n".join(json.dumps(j) for j in tw.ref_records(gen, rates, tk, seed))
        plan = [[int(x) for x in line.split()[:6]] for line in loader.ref_expand(text, 8, 164, 2048, 5).splitlines()]
        wcases.append({"gen": gen, "rates": list(rates), "template": tk, "seed": seed, "records": recs,
                       "plan": plan})
    with open(os.path.join(HERE, "workload_golden.json"), "w") as f:
        json.dump({"source": out["source"], "cases": wcases}, f)
    print("wrote", len(wcases), "workload cases")
    # per-vctx transcripts / logical progress of the reference simulator on a
    # two-job trace (integer bookkeeping the GPU engine must reproduce)
    import test_transcript_parity as tp  # noqa: E402
    sc, _ = tp.scenario()
    out = json.loads(loader.ref_simulate(json.dumps(sc)))
    # the event log of the same run (capture_log): per-vctx first-start /
    # finish streams and the field names of every kind (log schema)
    out_log = json.loads(loader.ref_simulate(json.dumps(dict(sc, capture_log=True))))
    streams, schema = tp.log_projection(out_log["event_log"])
    with open(os.path.join(HERE, "transcript_golden.json"), "w") as f:
        json.dump({"source": out_src(out), "scenario": sc, "transcripts": out["transcripts"],
                   "logical_progress": out["logical_progress"], "kernels_completed": out["kernels_completed"],
                   "log_streams": streams, "log_schema": schema}, f)
    print("wrote transcript golden:", out["kernels_completed"], "kernels")


def out_src(out):
    return "oracle/_ref SimEngine::simulate (reference corosim compiled from /root/reference)"


if __name__ == "__main__":
    main()
