"""CPU ORACLE — test infrastructure only, never on the product path.

Exact-rational restatement of the reference determinism lab (corosim numlab),
used by tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline leg
as the *checker* for the GPU reduction tenant.  Only those three may import it.

Parity pinning: validated against (1) the SPEC golden vectors
(SPEC.md:391-402), (2) the exhaustive n<=12 exact rounding-sequence property
 and (3) the reference library itself compiled from
/root/reference with a GMP-backed Boost shim (oracle/_ref, see oracle/Makefile
and tests/test_oracle_ref.py).

Each function cites the reference code it restates.
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from typing import List, Optional, Sequence

# ---------------------------------------------------------------------------
# mt19937_64 (std::mt19937_64, standard-mandated sequence) — rng.hpp:11-27
# ---------------------------------------------------------------------------
_MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 exactly (used by Rng, rng.hpp:13)."""

    n, m = 312, 156
    matrix_a = 0xB5026F5AA96619E9
    upper = 0xFFFFFFFF80000000
    lower = 0x7FFFFFFF

    def __init__(self, seed: int):
        mt = [0] * self.n
        mt[0] = seed & _MASK64
        for i in range(1, self.n):
            prev = mt[i - 1]
            mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & _MASK64
        self.mt = mt
        self.idx = self.n

    def _twist(self) -> None:
        mt, n, m = self.mt, self.n, self.m
        for i in range(n):
            x = (mt[i] & self.upper) | (mt[(i + 1) % n] & self.lower)
            xa = x >> 1
            if x & 1:
                xa ^= self.matrix_a
            mt[i] = mt[(i + m) % n] ^ xa
        self.idx = 0

    def next_u64(self) -> int:
        if self.idx >= self.n:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK64


class Rng:
    """Rng with explicit output transforms — rng.hpp:11-27."""

    def __init__(self, seed: int):
        self.gen = MT19937_64(seed)

    def next_u64(self) -> int:
        return self.gen.next_u64()

    def uniform01_fraction(self) -> Fraction:
        # (gen() >> 11) * 2^-53 is exact in double (rng.hpp:18)
        return Fraction(self.gen.next_u64() >> 11, 1 << 53)

    def uniform_fraction(self, lo: int = -1, hi: int = 1) -> Fraction:
        # lo + (hi - lo) * u ; for (lo, hi) = (-1, 1) the double arithmetic is
        # exact: 2*u is exact and -1 + 2u is a multiple of 2^-52 in (-1, 1).
        u = self.uniform01_fraction()
        return Fraction(lo) + Fraction(hi - lo) * u


# ---------------------------------------------------------------------------
# Float formats — float_format.hpp:18-57, float_format.cpp:24-78
# ---------------------------------------------------------------------------
FP16, BF16, FP32 = "fp16", "bf16", "fp32"
_LAYOUT = {FP16: (5, 10), BF16: (8, 7), FP32: (8, 23)}  # float_format.cpp:24-30


@dataclass(frozen=True)
class FloatValue:
    """FloatValue (float_format.hpp:35-50): finite exact rational or +/-inf/nan."""

    cls: str  # "finite" | "+inf" | "-inf" | "nan"
    value: Fraction = Fraction(0)

    @staticmethod
    def finite(v: Fraction) -> "FloatValue":
        return FloatValue("finite", Fraction(v))

    def is_finite(self) -> bool:
        return self.cls == "finite"

    def __eq__(self, other) -> bool:  # float_format.hpp:45-48
        if not isinstance(other, FloatValue):
            return NotImplemented
        if self.cls != other.cls:
            return False
        return self.cls != "finite" or self.value == other.value

    def __hash__(self):
        return hash((self.cls, self.value if self.cls == "finite" else 0))


def _floor_log2_abs(x: Fraction) -> int:
    """rational.cpp:121-135."""
    num, den = abs(x.numerator), x.denominator
    e = num.bit_length() - den.bit_length()

    def at_least(k: int) -> bool:
        return num >= (den << k) if k >= 0 else (num << -k) >= den

    if not at_least(e):
        e -= 1
    if at_least(e + 1):
        e += 1
    return e


def _pow2(e: int) -> Fraction:
    return Fraction(1 << e) if e >= 0 else Fraction(1, 1 << -e)


def max_finite(fmt: str) -> Fraction:
    eb, fb = _LAYOUT[fmt]
    bias = (1 << (eb - 1)) - 1
    return (2 - _pow2(-fb)) * _pow2(bias)  # float_format.cpp:32-35


def quantum(fmt: str, exp: int) -> Fraction:
    eb, fb = _LAYOUT[fmt]
    bias = (1 << (eb - 1)) - 1
    min_normal = 1 - bias
    e = min_normal if exp < min_normal else exp
    return _pow2(e - fb)  # float_format.cpp:37-40


def round_to(fmt: str, real: Fraction) -> FloatValue:
    """RNE ties-to-even with subnormals, overflow -> inf, no signed zero.

    float_format.cpp:43-67.
    """
    real = Fraction(real)
    if real == 0:
        return FloatValue.finite(Fraction(0))
    neg = real < 0
    mag = -real if neg else real
    q = quantum(fmt, _floor_log2_abs(mag))
    scaled = mag / q
    units, rem = divmod(scaled.numerator, scaled.denominator)
    twice = rem * 2
    if twice > scaled.denominator or (twice == scaled.denominator and (units & 1)):
        units += 1
    rounded = units * q
    if rounded > max_finite(fmt):
        return FloatValue("-inf" if neg else "+inf")
    return FloatValue.finite(-rounded if neg else rounded)


def add_rounded(fmt: str, a: FloatValue, b: FloatValue) -> FloatValue:
    """float_format.cpp:69-78."""
    if a.cls == "nan" or b.cls == "nan":
        return FloatValue("nan")
    if not a.is_finite() or not b.is_finite():
        if a.is_finite():
            return b
        if b.is_finite():
            return a
        return a if a.cls == b.cls else FloatValue("nan")
    return round_to(fmt, a.value + b.value)


# ---------------------------------------------------------------------------
# Reduction plans — reduction.cpp:7-71
# ---------------------------------------------------------------------------
def balanced_bounds(n: int, g: int) -> List[int]:
    """ReductionPlan::balanced (reduction.cpp:7-18): bound_i = floor(i*n/g)."""
    if n < 0 or g < 1:
        raise ValueError("PlanMismatch: balanced plan needs n >= 0 and splits >= 1")
    return [i * n // g for i in range(g + 1)]


def _fold(values: Sequence[FloatValue], fmt: str) -> FloatValue:
    """reduction.cpp:22-34: left-to-right, seeded with the first element."""
    acc = FloatValue.finite(Fraction(0))
    first = True
    for v in values:
        if first:
            acc, first = v, False
        else:
            acc = add_rounded(fmt, acc, v)
    return acc


def _combine_tree(partials: List[FloatValue], fmt: str) -> FloatValue:
    """reduction.cpp:36-48."""
    if not partials:
        return FloatValue.finite(Fraction(0))
    while len(partials) > 1:
        nxt = [add_rounded(fmt, partials[i], partials[i + 1]) for i in range(0, len(partials) - 1, 2)]
        if len(partials) % 2 == 1:
            nxt.append(partials[-1])
        partials = nxt
    return partials[0]


def reduce_with_plan(values: Sequence[FloatValue], fmt: str, bounds: Sequence[int],
                     tree_combine: bool = False) -> FloatValue:
    """reduction.cpp:52-71."""
    if len(bounds) < 2 or bounds[0] != 0 or bounds[-1] != len(values):
        raise ValueError("PlanMismatch: chunk bounds do not partition the input")
    partials = []
    for c in range(len(bounds) - 1):
        lo, hi = bounds[c], bounds[c + 1]
        if hi < lo:
            raise ValueError("PlanMismatch: descending chunk bound")
        partials.append(_fold(values[lo:hi], fmt))
    if tree_combine:
        return _combine_tree(partials, fmt)
    return _fold(partials, fmt)


def coupling_delta(values, fmt, bounds_i, bounds_j):
    """reduction.cpp:73-90 -> (bit_identical, finite, delta)."""
    a = reduce_with_plan(values, fmt, bounds_i)
    b = reduce_with_plan(values, fmt, bounds_j)
    same = a == b
    if a.is_finite() and b.is_finite():
        return same, True, abs(a.value - b.value)
    return same, same, Fraction(0)


# ---------------------------------------------------------------------------
# Seeded inputs and the reduction kernel's result — equivalence.cpp:7-25
# ---------------------------------------------------------------------------
def seeded_values(seed: int, n: int, fmt: str) -> List[FloatValue]:
    """equivalence.cpp:7-17: Rng(seed).uniform(-1,1) rounded into the format."""
    rng = Rng(seed)
    return [round_to(fmt, rng.uniform_fraction(-1, 1)) for _ in range(n)]


def reduction_result(seed: int, n: int, fmt: str, executed_grid: int) -> FloatValue:
    """equivalence.cpp:19-25."""
    g = executed_grid if executed_grid >= 1 else 1
    return reduce_with_plan(seeded_values(seed, n, fmt), fmt, balanced_bounds(n, g))


# ---------------------------------------------------------------------------
# Bit encodings (for comparing with native GPU results)
# ---------------------------------------------------------------------------
def encode_bits(fmt: str, v: FloatValue) -> int:
    """Encode an emulated value into its IEEE bit pattern (+0 for zero)."""
    eb, fb = _LAYOUT[fmt]
    width = 1 + eb + fb
    sign_bit = 1 << (width - 1)
    exp_all = ((1 << eb) - 1) << fb
    if v.cls == "nan":
        return exp_all | (1 << (fb - 1))
    if v.cls == "+inf":
        return exp_all
    if v.cls == "-inf":
        return sign_bit | exp_all
    x = v.value
    if x == 0:
        return 0
    sign = sign_bit if x < 0 else 0
    mag = -x if x < 0 else x
    bias = (1 << (eb - 1)) - 1
    e = _floor_log2_abs(mag)
    if e < 1 - bias:  # subnormal
        m = mag / _pow2(1 - bias - fb)
        assert m.denominator == 1
        return sign | int(m)
    m = mag / _pow2(e - fb)
    assert m.denominator == 1
    return sign | ((e + bias) << fb) | (int(m) - (1 << fb))


def decode_bits(fmt: str, bits: int) -> FloatValue:
    eb, fb = _LAYOUT[fmt]
    width = 1 + eb + fb
    sign = -1 if bits >> (width - 1) & 1 else 1
    e = (bits >> fb) & ((1 << eb) - 1)
    m = bits & ((1 << fb) - 1)
    bias = (1 << (eb - 1)) - 1
    if e == (1 << eb) - 1:
        if m:
            return FloatValue("nan")
        return FloatValue("+inf" if sign > 0 else "-inf")
    if e == 0:
        return FloatValue.finite(sign * m * _pow2(1 - bias - fb))
    return FloatValue.finite(sign * ((1 << fb) + m) * _pow2(e - bias - fb))


def seeded_bits(seed: int, n: int, fmt: str) -> List[int]:
    return [encode_bits(fmt, v) for v in seeded_values(seed, n, fmt)]


def exact_sequence_oracle(values: Sequence[FloatValue], fmt: str, bounds: Sequence[int]) -> FloatValue:
    """Independent golden rounding-sequence oracle: walks
    the same addition sequence but re-derives every rounding from the bit
    grid (enumerating the two neighbouring representable values), not from
    round_to's quantum arithmetic."""

    def nearest(x: Fraction) -> FloatValue:
        if x == 0:
            return FloatValue.finite(Fraction(0))
        neg = x < 0
        mag = -x if neg else x
        # binary search over non-negative finite bit patterns (monotone)
        eb, fb = _LAYOUT[fmt]
        top = (((1 << eb) - 1) << fb) - 1  # max finite pattern
        lo, hi = 0, top
        if mag >= decode_bits(fmt, top).value:
            below = top
        else:
            while lo < hi:
                mid = (lo + hi + 1) // 2
                if decode_bits(fmt, mid).value <= mag:
                    lo = mid
                else:
                    hi = mid - 1
            below = lo
        vb = decode_bits(fmt, below).value
        if vb == mag:
            res = vb
        else:
            above = below + 1
            va = decode_bits(fmt, above).value if above <= top else None
            if va is None:
                # beyond max finite: overflow boundary is max + half ulp of top binade
                ulp = decode_bits(fmt, top).value - decode_bits(fmt, top - 1).value
                limit = vb + ulp / 2
                if mag > limit or (mag == limit and (below & 1)):
                    return FloatValue("-inf" if neg else "+inf")
                res = vb
            else:
                d_lo, d_hi = mag - vb, va - mag
                if d_lo < d_hi or (d_lo == d_hi and below % 2 == 0):
                    res = vb
                else:
                    res = va
                    if above == top + 1:
                        return FloatValue("-inf" if neg else "+inf")
        return FloatValue.finite(-res if neg else res)

    def add(a: FloatValue, b: FloatValue) -> FloatValue:
        if not (a.is_finite() and b.is_finite()):
            return add_rounded(fmt, a, b)
        return nearest(a.value + b.value)

    partials = []
    for c in range(len(bounds) - 1):
        chunk = values[bounds[c]:bounds[c + 1]]
        acc: Optional[FloatValue] = None
        for v in chunk:
            acc = v if acc is None else add(acc, v)
        partials.append(acc if acc is not None else FloatValue.finite(Fraction(0)))
    acc = None
    for p in partials:
        acc = p if acc is None else add(acc, p)
    return acc if acc is not None else FloatValue.finite(Fraction(0))
