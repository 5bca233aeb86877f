"""The product's native determinism-lab inputs (csrc/numlab.cpp:
ds_seeded_values, ds_round_to — SURVEY 8a rows a20/a21) against the
reference's golden vectors (tests/golden/round_to_golden.json, produced by the
reference library) and the oracle's independent C restatement
(oracle/cnumlab.c) on seeded streams and random doubles across the full
exponent range (subnormals, overflow, ties).  Also add_normalization
(metrics.cpp:81-102).  CPU only."""
import ctypes
import json
import math
import os
import random
from fractions import Fraction

import pytest

from oracle import loader
from paper_2603_15042_b200 import runtime as rt

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "round_to_golden.json")
FMT = {"fp16": 0, "bf16": 1, "fp32": 2}


def test_round_to_reference_golden():
    cases = json.load(open(GOLDEN))["cases"]
    n = 0
    for c in cases:
        x = Fraction(c["num"], c["den"])
        if x.denominator & (x.denominator - 1) or abs(x.numerator) >= 2 ** 53:
            continue  # not exactly a double: the lab's inputs always are
        assert rt.round_to(FMT[c["fmt"]], float(x)) == c["bits"], c
        n += 1
    assert n >= 10
    # SPEC.md:391-393
    assert rt.round_to(0, 1.0) == 0x3C00
    assert rt.round_to(0, 1 + 2 ** -11) == 0x3C00
    assert rt.round_to(1, 1 + 2 ** -8) == 0x3F80


@pytest.mark.parametrize("fmt", [0, 1, 2])
def test_round_to_matches_oracle_on_random_doubles(fmt):
    cn = loader.cnumlab()
    rng = random.Random(1234 + fmt)
    for _ in range(60000):
        e = rng.randint(-160, 140)
        m = rng.getrandbits(53) | (1 << 52) if rng.random() < 0.9 else rng.getrandbits(rng.randint(1, 12))
        x = math.ldexp(m, e - 52) * (-1 if rng.random() < 0.5 else 1)
        if x == 0 or math.isinf(x):
            continue
        assert rt.round_to(fmt, x) == cn.cn_round_double(fmt, x), (fmt, x.hex())
    # exact ties around every binade of the format (half a quantum up from a
    # representable value): ties-to-even
    for k in range(-30, 20):
        for frac in (1, 3, 5, 255):
            x = math.ldexp(1 + frac * 2.0 ** -12, k)
            assert rt.round_to(fmt, x) == cn.cn_round_double(fmt, x), (fmt, x.hex())


@pytest.mark.parametrize("fmt", [0, 1, 2])
def test_seeded_values_match_oracle(fmt):
    cn = loader.cnumlab()
    for seed in (0, 1, 7, 12345, 2 ** 63 + 5):
        n = 4096
        want = (ctypes.c_uint32 * n)()
        cn.cn_seeded_bits(seed, n, fmt, want)
        assert rt.seeded_values(seed, n, fmt) == list(want), seed


def test_add_normalization():
    # job 0: solo 10 ns over a shared span of 40 -> 1/4; job 1: equal spans -> 1;
    # job 2: missing shared span -> 0; job 3: empty shared span -> 0
    norm, agg = rt.add_normalization([(0, 40), (5, 15), None, (7, 7)], [(0, 10), (0, 10), (0, 3), (0, 3)])
    assert norm == [Fraction(1, 4), Fraction(1), Fraction(0), Fraction(0)]
    assert agg == pytest.approx(1.25)
