// Native input stream of the reduction tenant: the reference determinism
// lab's seeded_values (proj/src/numlab/equivalence.cpp:7-17) —
// Rng(seed).uniform(-1, 1) (rng.hpp:18-21: lo + (hi - lo) * ((u64 >> 11) *
// 2^-53), an exact double) rounded once, ties-to-even, into the target
// format with subnormals, overflow to infinity and no signed zero
// (round_to, float_format.cpp:43-67).
//
// The rounding works on the double's bit fields: the 53-bit significand is
// shifted to the target's quantum at its exponent (the subnormal quantum
// below the normal range) and rounded half-to-even on the dropped bits.
#include <cstdint>
#include <cstring>
#include <random>

#include "../../include/detshare/ds.h"

namespace {

struct Layout {
    int eb, fb;  // exponent / fraction bits: fp16 (5, 10), bf16 (8, 7), fp32 (8, 23)
};

bool layout_of(int fmt, Layout* l) {
    switch (fmt) {
        case 0: *l = {5, 10}; return true;
        case 1: *l = {8, 7}; return true;
        case 2: *l = {8, 23}; return true;
    }
    return false;
}

uint32_t round_bits(const Layout& L, double x) {
    uint64_t d;
    std::memcpy(&d, &x, 8);
    const uint32_t sign = (uint32_t)(d >> 63) << (L.eb + L.fb);
    const int dexp = (int)((d >> 52) & 0x7ff);
    uint64_t sig = d & ((1ull << 52) - 1);
    if (dexp == 0 && sig == 0) return 0u;  // +0 only
    if (dexp == 0x7ff) return sign | (((1u << L.eb) - 1u) << L.fb) | (sig ? 1u : 0u);
    int e;  // value = sig * 2^(e - 52), sig in [2^52, 2^53) for normal doubles
    if (dexp == 0) {  // double subnormal: normalise
        e = -1022;
        while (!(sig & (1ull << 52))) {
            sig <<= 1;
            --e;
        }
    } else {
        sig |= 1ull << 52;
        e = dexp - 1023;
    }
    const int bias = (1 << (L.eb - 1)) - 1;
    const int emin = 1 - bias;
    // drop bits down to the target quantum 2^(max(e, emin) - fb)
    const int shift = 52 - L.fb + (e < emin ? emin - e : 0);
    uint64_t units;
    if (shift >= 64) {
        units = 0;
    } else {
        units = sig >> shift;
        const uint64_t rem = sig & ((1ull << shift) - 1);
        const uint64_t half = 1ull << (shift - 1);
        if (rem > half || (rem == half && (units & 1))) ++units;
    }
    if (units == 0) return 0u;  // rounds to zero: +0 (no signed zero)
    if (e < emin) return sign | (uint32_t)units;  // subnormal (units == 2^fb encodes the min normal)
    if (units >> (L.fb + 1)) {  // carry into the next binade
        units >>= 1;
        ++e;
    }
    if (e > bias) return sign | (((1u << L.eb) - 1u) << L.fb);  // overflow -> infinity
    return sign | ((uint32_t)(e + bias) << L.fb) | (uint32_t)(units & ((1ull << L.fb) - 1));
}

}  // namespace

extern "C" {

int ds_round_to(int fmt, double x, uint32_t* bits) {
    Layout L;
    if (!bits || !layout_of(fmt, &L)) return DS_INVALID_ARGUMENT;
    *bits = round_bits(L, x);
    return DS_OK;
}

int ds_seeded_values(uint64_t seed, int64_t n, int fmt, uint32_t* bits) {
    Layout L;
    if ((!bits && n > 0) || n < 0 || !layout_of(fmt, &L)) return DS_INVALID_ARGUMENT;
    std::mt19937_64 gen(seed);  // Rng (rng.hpp:11-40)
    for (int64_t i = 0; i < n; ++i) {
        const double u = (double)(gen() >> 11) * 0x1.0p-53;
        bits[i] = round_bits(L, -1.0 + 2.0 * u);
    }
    return DS_OK;
}

}  // extern "C"
