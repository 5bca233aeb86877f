"""ctypes loaders for the compiled oracles (test infrastructure only).

``cnumlab()``  -> oracle/_build/libcnumlab.so   (fast C restatement)
``reference()`` -> oracle/_ref/libcorosim_ref.so (reference compiled here)
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from fractions import Fraction
from typing import Optional

from . import numlab as nl

HERE = os.path.dirname(os.path.abspath(__file__))
CN_PATH = os.path.join(HERE, "_build", "libcnumlab.so")
REF_PATH = os.path.join(HERE, "_ref", "libcorosim_ref.so")
REF_SRC = "/root/reference/proj"

FMT_CODE = {nl.FP16: 0, nl.BF16: 1, nl.FP32: 2}


def build(ref: bool = True) -> None:
    """Compile the C restatement and, when the reference tree is present,
    the reference library (oracle/Makefile)."""
    targets = ["cnumlab"]
    if ref and os.path.isdir(REF_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-j8", "-C", HERE] + targets, check=True)


_cn = None
_ref = None


def cnumlab():
    global _cn
    if _cn is None:
        if not os.path.exists(CN_PATH):
            build(ref=False)
        lib = ctypes.CDLL(CN_PATH)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        lib.cn_round_double.restype = ctypes.c_uint32
        lib.cn_round_double.argtypes = [ctypes.c_int, ctypes.c_double]
        lib.cn_add_bits.restype = ctypes.c_uint32
        lib.cn_add_bits.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32]
        lib.cn_seeded_bits.restype = None
        lib.cn_seeded_bits.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, u32p]
        lib.cn_reduce_bits.restype = ctypes.c_uint32
        lib.cn_reduce_bits.argtypes = [u32p, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.c_int]
        lib.cn_chunk_partials.restype = None
        lib.cn_chunk_partials.argtypes = [u32p, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, u32p]
        lib.cn_reduction_result.restype = ctypes.c_uint32
        lib.cn_reduction_result.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_int64]
        lib.cn_uniform_f32.restype = None
        lib.cn_uniform_f32.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                       ctypes.POINTER(ctypes.c_float)]
        lib.cn_u64_stream.restype = None
        lib.cn_u64_stream.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.POINTER(ctypes.c_uint64)]
        lib.cn_sgemm_fma.restype = None
        lib.cn_sgemm_fma.argtypes = [ctypes.POINTER(ctypes.c_float)] * 3 + [ctypes.c_int] * 5
        _cn = lib
    return _cn


def reference_available() -> bool:
    return os.path.exists(REF_PATH) or os.path.isdir(REF_SRC)


def reference():
    """The reference library compiled from /root/reference (None if neither
    the built .so nor the sources are present)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            if not os.path.isdir(REF_SRC):
                return None
            build(ref=True)
        lib = ctypes.CDLL(REF_PATH)
        for name in ("ref_reduction_result",):
            getattr(lib, name).argtypes = [ctypes.c_ulonglong, ctypes.c_longlong, ctypes.c_int,
                                           ctypes.c_longlong, ctypes.c_char_p, ctypes.c_long]
        lib.ref_seeded_value.argtypes = [ctypes.c_ulonglong, ctypes.c_longlong, ctypes.c_int,
                                         ctypes.c_longlong, ctypes.c_char_p, ctypes.c_long]
        lib.ref_round_to.argtypes = [ctypes.c_int, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p,
                                     ctypes.c_long]
        lib.ref_reduce_values.argtypes = [ctypes.c_int, ctypes.c_char_p, ctypes.c_longlong,
                                          ctypes.c_longlong, ctypes.c_int, ctypes.c_char_p, ctypes.c_long]
        lib.ref_simulate_json.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_long]
        lib.ref_equivalence_json.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_long]
        lib.ref_gen_trace.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double)] + [ctypes.c_int] * 7 + [
            ctypes.c_ulonglong, ctypes.c_char_p, ctypes.c_long]
        lib.ref_migration_set.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_char_p, ctypes.c_long]
        lib.ref_expand.argtypes = [ctypes.c_char_p, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong,
                                   ctypes.c_int, ctypes.c_char_p, ctypes.c_long]
        _ref = lib
    return _ref


def parse_fv(s: str) -> nl.FloatValue:
    if s == "inf":
        return nl.FloatValue("+inf")
    if s in ("-inf", "nan"):
        return nl.FloatValue(s)
    if s.startswith("error"):
        raise RuntimeError(s)
    a, b = s.split("/")
    return nl.FloatValue.finite(Fraction(int(a), int(b)))


def _call(fn, *args, cap: int = 1 << 20) -> str:
    buf = ctypes.create_string_buffer(cap)
    rc = fn(*args, buf, cap)
    out = buf.value.decode()
    if rc != 0:
        raise RuntimeError(f"reference call failed ({rc}): {out}")
    return out


def ref_reduction_result(seed: int, n: int, fmt: str, grid: int) -> nl.FloatValue:
    return parse_fv(_call(reference().ref_reduction_result, seed, n, FMT_CODE[fmt], grid))


def ref_round_to(fmt: str, x: Fraction) -> nl.FloatValue:
    return parse_fv(_call(reference().ref_round_to, FMT_CODE[fmt], str(x.numerator).encode(),
                          str(x.denominator).encode()))


def exact_decimal(x: Fraction) -> str:
    """Exact terminating decimal of a dyadic rational."""
    assert x.denominator & (x.denominator - 1) == 0
    neg = x < 0
    x = abs(x)
    k = x.denominator.bit_length() - 1
    digits = x.numerator * (5 ** k)
    s = str(digits).rjust(k + 1, "0")
    whole, frac = (s[:-k], s[-k:]) if k else (s, "")
    out = whole + ("." + frac if frac else "")
    return ("-" if neg else "") + out


def ref_reduce_values(fmt: str, values, g: int, tree: bool = False) -> nl.FloatValue:
    text = "\n".join(exact_decimal(v.value) for v in values).encode()
    return parse_fv(_call(reference().ref_reduce_values, FMT_CODE[fmt], text, len(values), g, int(tree)))


def ref_simulate(scenario_json: str) -> str:
    return _call(reference().ref_simulate_json, scenario_json.encode(), cap=1 << 26)


def ref_equivalence(scenario_json: str) -> str:
    return _call(reference().ref_equivalence_json, scenario_json.encode(), cap=1 << 20)


def ref_gen_trace(which: str, rates, kind: int, prompt: int, prompt_max: int, output: int, output_max: int,
                  iterations: int, streams: int, seed: int) -> str:
    """gen_poisson / gen_burst of the reference (trace.cpp:189-232) as JSONL."""
    arr = (ctypes.c_double * len(rates))(*rates)
    return _call(reference().ref_gen_trace, 0 if which == "poisson" else 1, arr, kind, prompt, prompt_max, output,
                 output_max, iterations, streams, seed, cap=1 << 26)


def ref_expand(trace_jsonl: str, tokens_per_grid_unit: int, decode_grid: int, train_grid: int,
               default_iterations: int) -> str:
    """expand_workload of the reference (workload.cpp:51-174), one line per kernel."""
    return _call(reference().ref_expand, trace_jsonl.encode(), tokens_per_grid_unit, decode_grid, train_grid,
                 default_iterations, cap=1 << 26)


def ref_migration_set(regions, touched, dst: int, full: bool = False) -> str:
    """compute_migration_set / full_eager_set of the reference (migration.cpp:21-58).
    regions: [(id, bytes, dirty, [places])]."""
    text = "\n".join(f"{i} {b} {int(d)} {','.join(map(str, p)) or '-'}" for i, b, d, p in regions)
    return _call(reference().ref_migration_set, text.encode(), " ".join(map(str, touched)).encode(), dst, int(full))


def ref_compute_metrics(outcomes, makespan: int, kernels_completed: int) -> dict:
    """compute_metrics of the reference (metrics.cpp:35-85) over outcomes
    [dict(inference, completed, output_tokens, has_slo, arrival, first, last,
    ttft_slo, tpot_slo, kernels_done)] with integer times; exact Fractions."""
    n = len(outcomes)
    I = lambda k: (ctypes.c_int * max(1, n))(*[int(o[k]) for o in outcomes])
    L = lambda k: (ctypes.c_longlong * max(1, n))(*[int(o[k]) for o in outcomes])
    text = _call(reference().ref_compute_metrics, ctypes.c_longlong(n), I("inference"), I("completed"),
                 I("output_tokens"), I("has_slo"), L("arrival"), L("first"), L("last"), L("ttft_slo"),
                 L("tpot_slo"), L("kernels_done"), ctypes.c_longlong(makespan), ctypes.c_longlong(kernels_completed))
    out = {}
    for line in text.splitlines():
        k, v = line.split()
        out[k] = Fraction(v) if "/" in v else int(v)
    return out
