/*
 * CPU ORACLE — test infrastructure only (tests/, __graft_entry__.smoke(),
 * bench.py's cpu_baseline leg).  Never linked into or called by the product.
 *
 * Fast C restatement of the reference determinism lab for large n, plus the
 * fixed-order FP32 SGEMM checker for the SGEMM tenant.
 *
 *   rng.hpp:11-27             mt19937_64 + uniform(-1,1) transform
 *   float_format.cpp:43-67    round_to: RNE ties-to-even, subnormals, overflow
 *                             to +/-inf, no signed zero
 *   float_format.cpp:69-78    add_rounded: exact sum, one rounding
 *   reduction.cpp:7-71        balanced plan, left-to-right fold, sequential or
 *                             pairwise-tree combine
 *   equivalence.cpp:7-25      seeded_values / reduction_result
 *
 * Exactness argument: every value of fp16/bf16/fp32 is a double; the exact
 * sum of two such values rounded once to double and then once to the target
 * is the correctly rounded target sum because double has p' = 53 >= 2p + 1
 * for p in {11, 8, 24} and covers the targets' exponent ranges (subnormals
 * included) with normal doubles.  Parity is additionally pinned against the
 * exact-rational Python restatement (oracle/numlab.py) and the reference
 * library itself (oracle/_ref) in tests/test_oracle_*.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------- mt19937_64 ---------------- */
typedef struct {
    uint64_t mt[312];
    int idx;
} cn_mt64;

static void mt_seed(cn_mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i) {
        uint64_t p = s->mt[i - 1];
        s->mt[i] = 6364136223846793005ULL * (p ^ (p >> 62)) + (uint64_t)i;
    }
    s->idx = 312;
}

static uint64_t mt_next(cn_mt64* s) {
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t y = s->mt[s->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* Rng::uniform(lo, hi) = lo + (hi-lo) * ((gen()>>11) * 2^-53)  (rng.hpp:18-21) */
static double rng_uniform(cn_mt64* s, double lo, double hi) {
    double u = (double)(mt_next(s) >> 11) * 0x1.0p-53;
    return lo + (hi - lo) * u;
}

/* ---------------- formats ---------------- */
enum { CN_FP16 = 0, CN_BF16 = 1, CN_FP32 = 2 }; /* FloatFormatKind order */

static void layout(int fmt, int* eb, int* fb) {
    if (fmt == CN_FP16) { *eb = 5; *fb = 10; }
    else if (fmt == CN_BF16) { *eb = 8; *fb = 7; }
    else { *eb = 8; *fb = 23; }
}

/* Correctly round a finite double into the format (RNE, subnormals,
 * overflow -> inf, zero -> +0).  Returns the raw bit pattern. */
static uint32_t round_double(int fmt, double x) {
    int eb, fb;
    layout(fmt, &eb, &fb);
    int width = 1 + eb + fb;
    uint32_t sign = (x < 0) ? (1u << (width - 1)) : 0u;
    double mag = fabs(x);
    if (mag == 0.0) return 0u; /* no signed zero (float_format.cpp:44) */
    int bias = (1 << (eb - 1)) - 1;
    int e2;
    double fr = frexp(mag, &e2); /* mag = fr * 2^e2, fr in [0.5,1) */
    int64_t m = (int64_t)ldexp(fr, 53); /* mag = m * 2^(e2-53) exactly */
    int mexp = e2 - 53;
    int floor_log2 = e2 - 1;
    int min_normal = 1 - bias;
    int qe = (floor_log2 < min_normal ? min_normal : floor_log2) - fb; /* quantum exponent */
    int shift = qe - mexp;
    int64_t units;
    if (shift <= 0) {
        units = m << (-shift); /* exact (cannot overflow: result < 2^(fb+2)) */
    } else if (shift > 60) {
        units = 0; /* m < 2^53 < half quantum */
    } else {
        units = m >> shift;
        int64_t rem = m & ((1LL << shift) - 1);
        int64_t half = 1LL << (shift - 1);
        if (rem > half || (rem == half && (units & 1))) units += 1;
    }
    if (units == 0) return 0u; /* rounds to zero: +0 */
    /* encode units * 2^qe */
    uint32_t exp_all = ((1u << eb) - 1u) << fb;
    if (qe == min_normal - fb && units < (1LL << fb)) {
        return sign | (uint32_t)units; /* subnormal */
    }
    /* normalise: units in [2^fb, 2^(fb+1)] (2^(fb+1) after carry) */
    int e = qe + fb;
    if (units >= (1LL << (fb + 1))) { units >>= 1; e += 1; }
    if (e > bias) return sign | exp_all; /* overflow -> inf */
    return sign | ((uint32_t)(e + bias) << fb) | ((uint32_t)units - (1u << fb));
}

/* Decode bits; returns class: 0 finite, 1 +inf, 2 -inf, 3 nan. */
static int decode(int fmt, uint32_t bits, double* out) {
    int eb, fb;
    layout(fmt, &eb, &fb);
    int width = 1 + eb + fb;
    int neg = (bits >> (width - 1)) & 1;
    uint32_t e = (bits >> fb) & ((1u << eb) - 1u);
    uint32_t m = bits & ((1u << fb) - 1u);
    int bias = (1 << (eb - 1)) - 1;
    if (e == (1u << eb) - 1u) {
        if (m) return 3;
        return neg ? 2 : 1;
    }
    double v = (e == 0) ? ldexp((double)m, 1 - bias - fb) : ldexp((double)((1u << fb) + m), (int)e - bias - fb);
    *out = neg ? -v : v;
    return 0;
}

static uint32_t nan_bits(int fmt) {
    int eb, fb;
    layout(fmt, &eb, &fb);
    return (((1u << eb) - 1u) << fb) | (1u << (fb - 1));
}

/* add_rounded (float_format.cpp:69-78) on bit patterns */
static uint32_t add_bits(int fmt, uint32_t a, uint32_t b) {
    double x = 0, y = 0;
    int ca = decode(fmt, a, &x), cb = decode(fmt, b, &y);
    if (ca == 3 || cb == 3) return nan_bits(fmt);
    if (ca != 0 || cb != 0) {
        if (ca == 0) return b;
        if (cb == 0) return a;
        return ca == cb ? a : nan_bits(fmt);
    }
    return round_double(fmt, x + y);
}

static uint32_t fold(int fmt, const uint32_t* v, int64_t n) {
    if (n <= 0) return 0u; /* FloatValue::finite(0) */
    uint32_t acc = v[0];
    for (int64_t i = 1; i < n; ++i) acc = add_bits(fmt, acc, v[i]);
    return acc;
}

/* ---------------- exported API ---------------- */
uint32_t cn_round_double(int fmt, double x) { return round_double(fmt, x); }

uint32_t cn_add_bits(int fmt, uint32_t a, uint32_t b) { return add_bits(fmt, a, b); }

void cn_seeded_bits(uint64_t seed, int64_t n, int fmt, uint32_t* out) {
    cn_mt64 s;
    mt_seed(&s, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = round_double(fmt, rng_uniform(&s, -1.0, 1.0));
}

void cn_u64_stream(uint64_t seed, int64_t n, uint64_t* out) {
    cn_mt64 s;
    mt_seed(&s, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = mt_next(&s);
}

/* reduce_with_plan with ReductionPlan::balanced(n, g) (reduction.cpp:7-71) */
uint32_t cn_reduce_bits(const uint32_t* bits, int64_t n, int fmt, int64_t g, int tree) {
    if (g < 1) g = 1;
    uint32_t* partials = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)g);
    for (int64_t c = 0; c < g; ++c) {
        int64_t lo = c * n / g, hi = (c + 1) * n / g;
        partials[c] = fold(fmt, bits + lo, hi - lo);
    }
    uint32_t r;
    if (!tree) {
        r = fold(fmt, partials, g);
    } else {
        int64_t m = g;
        while (m > 1) {
            int64_t k = 0;
            for (int64_t i = 0; i + 1 < m; i += 2) partials[k++] = add_bits(fmt, partials[i], partials[i + 1]);
            if (m % 2 == 1) partials[k++] = partials[m - 1];
            m = k;
        }
        r = partials[0];
    }
    free(partials);
    return r;
}

/* Chunk partials only (what logical block c of the reduction tenant writes). */
void cn_chunk_partials(const uint32_t* bits, int64_t n, int fmt, int64_t g, uint32_t* out) {
    for (int64_t c = 0; c < g; ++c) {
        int64_t lo = c * n / g, hi = (c + 1) * n / g;
        out[c] = fold(fmt, bits + lo, hi - lo);
    }
}

/* reduction_result (equivalence.cpp:19-25) */
uint32_t cn_reduction_result(uint64_t seed, int64_t n, int fmt, int64_t g) {
    uint32_t* v = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
    cn_seeded_bits(seed, n, fmt, v);
    uint32_t r = cn_reduce_bits(v, n, fmt, g, 0);
    free(v);
    return r;
}

/* Rng(seed).uniform(lo,hi) rounded (RNE) to float: SGEMM tenant inputs. */
void cn_uniform_f32(uint64_t seed, int64_t n, double lo, double hi, float* out) {
    cn_mt64 s;
    mt_seed(&s, seed);
    for (int64_t i = 0; i < n; ++i) {
        uint32_t b = round_double(CN_FP32, rng_uniform(&s, lo, hi));
        memcpy(&out[i], &b, 4);
    }
}

/* C[M,N] = A[M,K] . B[K,N], row-major; per element a k-ascending fmaf chain
 * seeded with +0 — the fixed arithmetic order of the SGEMM tenant body. */
void cn_sgemm_fma(const float* A, const float* B, float* C, int M, int N, int K, int row_begin, int row_end) {
    if (row_end > M) row_end = M;
    for (int i = row_begin; i < row_end; ++i) {
        for (int j = 0; j < N; ++j) {
            float acc = 0.0f;
            for (int k = 0; k < K; ++k) acc = fmaf(A[(size_t)i * K + k], B[(size_t)k * N + j], acc);
            C[(size_t)i * N + j] = acc;
        }
    }
}
