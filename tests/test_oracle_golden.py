"""Pin the oracle restatements (oracle/numlab.py exact-rational, oracle/cnumlab.c
fast) against the SPEC golden vectors and against
the committed fixtures generated from the reference library itself
(tests/golden/make_golden.py)."""
import ctypes
import json
import os
import random
from fractions import Fraction as F

import pytest

from oracle import loader, numlab as nl

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def fv(x):
    return nl.FloatValue.finite(F(x))


# -- SPEC.md:391-393 round_to examples ---------------------------------------
def test_round_to_spec_examples():
    assert nl.round_to(nl.FP16, F(1)) == fv(1)
    assert nl.round_to(nl.FP16, 1 + F(1, 2**11)) == fv(1)  # tie -> even
    assert nl.round_to(nl.BF16, 1 + F(1, 2**8)) == fv(1)


def test_round_to_no_signed_zero_and_overflow():
    assert nl.round_to(nl.FP16, -F(1, 2**26)) == fv(0)
    assert nl.encode_bits(nl.FP16, nl.round_to(nl.FP16, -F(1, 2**26))) == 0
    assert nl.round_to(nl.FP16, F(65520)).cls == "+inf"  # max + half ulp ties up
    assert nl.round_to(nl.FP16, F(65519)) == fv(65504)
    assert nl.round_to(nl.FP16, -F(70000)).cls == "-inf"


# -- SPEC.md:400-402 reduce_with_plan examples --------------------------------
def test_reduce_spec_examples():
    vals = [fv(1), fv(F(1, 2**11)), fv(F(1, 2**11))]
    assert nl.reduce_with_plan(vals, nl.FP16, nl.balanced_bounds(3, 1)) == fv(1)
    assert nl.reduce_with_plan(vals, nl.FP16, nl.balanced_bounds(3, 3)) == fv(1)
    # balanced(3,2) = {0,1,3}: chunks [1], [2^-11, 2^-11] -> 1 + 2^-10 (reduction.cpp:14-16)
    assert nl.reduce_with_plan(vals, nl.FP16, nl.balanced_bounds(3, 2)) == fv(1 + F(1, 2**10))
    same, fin, d = nl.coupling_delta(vals, nl.FP16, nl.balanced_bounds(3, 1), nl.balanced_bounds(3, 2))
    assert not same and fin and d == F(1, 2**10)
    bvals = [fv(1), fv(F(1, 2**8)), fv(F(1, 2**8))]
    assert nl.reduce_with_plan(bvals, nl.BF16, nl.balanced_bounds(3, 2)) == fv(F(1009, 1000) - F(1009, 1000) + F(129, 128))


def test_fp32_fixed_plan_deterministic(cn):
    a = cn.cn_reduction_result(5, 4096, 2, 1)
    b = cn.cn_reduction_result(5, 4096, 2, 1)
    assert a == b


# -- SPEC.md:613 exact-rational rounding-sequence oracle, n <= 12 -------------
@pytest.mark.parametrize("fmt", [nl.FP16, nl.BF16, nl.FP32])
def test_exhaustive_small_n_vs_sequence_oracle(fmt):
    rnd = random.Random(1234)
    for n in range(1, 13):
        for _ in range(6):
            vals = [nl.round_to(fmt, F(rnd.randint(-2**20, 2**20), 2**rnd.randint(8, 22))) for _ in range(n)]
            for g in range(1, n + 1):
                b = nl.balanced_bounds(n, g)
                assert nl.reduce_with_plan(vals, fmt, b) == nl.exact_sequence_oracle(vals, fmt, b)


# -- C restatement == exact-rational restatement -------------------------------
@pytest.mark.parametrize("fmt", [nl.FP16, nl.BF16, nl.FP32])
def test_cnumlab_matches_fraction_oracle(cn, fmt):
    code = loader.FMT_CODE[fmt]
    for seed in range(3):
        n = 700
        vals = nl.seeded_values(seed, n, fmt)
        bits = (ctypes.c_uint32 * n)()
        cn.cn_seeded_bits(seed, n, code, bits)
        assert list(bits) == [nl.encode_bits(fmt, v) for v in vals]
        for g in (1, 2, 5, 64, 699, 700, 900):
            want = nl.encode_bits(fmt, nl.reduce_with_plan(vals, fmt, nl.balanced_bounds(n, g)))
            assert cn.cn_reduce_bits(bits, n, code, g, 0) == want
        want_t = nl.encode_bits(fmt, nl.reduce_with_plan(vals, fmt, nl.balanced_bounds(n, 13), True))
        assert cn.cn_reduce_bits(bits, n, code, 13, 1) == want_t


def test_cnumlab_round_double_random(cn):
    rnd = random.Random(7)
    for fmt in (nl.FP16, nl.BF16, nl.FP32):
        code = loader.FMT_CODE[fmt]
        for _ in range(3000):
            x = rnd.uniform(-1, 1) * 2.0 ** rnd.randint(-160, 140)
            want = nl.encode_bits(fmt, nl.round_to(fmt, F(x)))
            assert cn.cn_round_double(code, x) == want, (fmt, x)


# -- committed fixtures from the reference library ----------------------------
def test_reduction_golden_fixture(cn):
    data = json.load(open(os.path.join(GOLDEN, "reduction_golden.json")))
    for c in data["cases"]:
        n = c.get("n", data["n"])
        got = cn.cn_reduction_result(c["seed"], n, loader.FMT_CODE[c["fmt"]], c["grid"])
        assert got == c["bits"], c


def test_round_to_golden_fixture():
    data = json.load(open(os.path.join(GOLDEN, "round_to_golden.json")))
    for c in data["cases"]:
        got = nl.round_to(c["fmt"], F(c["num"], c["den"]))
        assert got.cls == c["cls"] and nl.encode_bits(c["fmt"], got) == c["bits"], c


# -- SPEC.md:611 Eq. 1 dichotomy (scaled to a CPU-test budget) -----------------
def test_eq1_dichotomy(cn):
    import statistics
    n, seeds = 4096, 200
    d16, d_bf = [], []
    nz = 0
    for s in range(seeds):
        a = cn.cn_reduction_result(s, n, 0, 1)
        b = cn.cn_reduction_result(s, n, 0, 64)
        x, y = nl.decode_bits(nl.FP16, a).value, nl.decode_bits(nl.FP16, b).value
        nz += x != y
        d16.append(abs(x - y))
        a = cn.cn_reduction_result(s, n, 1, 1)
        b = cn.cn_reduction_result(s, n, 1, 64)
        d_bf.append(abs(nl.decode_bits(nl.BF16, a).value - nl.decode_bits(nl.BF16, b).value))
    # SPEC.md:611 asks for >= 99%; the reference itself yields 976/1000 over
    # seeds 0..999 (checked three ways: oracle/_ref, numlab.py, cnumlab.c), so
    # the pinned property is the reference's own rate, not the SPEC's target.
    assert nz >= 0.95 * seeds
    assert statistics.median(d_bf) >= 5 * statistics.median(d16)
