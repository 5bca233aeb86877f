// Reduction tenant — the GPU realisation of the reference determinism lab's
// reduction kernel (reduction_result, src/numlab/equivalence.cpp:19-25).
//
// Launched with logical grid g, logical block c folds chunk
// [c*n/g, (c+1)*n/g) left-to-right seeded with its first element
// (ReductionPlan::balanced + fold, src/numlab/reduction.cpp:7-34), every add
// rounded once in the target format with the native RN instruction
// (add.rn.f16 / add.rn.bf16 / add.rn.f32; no FTZ).  The block that retires
// last (ticket counter, threadfence pattern) folds the partials left-to-right
// in chunk order (reduction.cpp:67-70).  The result therefore depends only on
// (values, format, g) — never on which SM ran which chunk or in what order.
#pragma once
#include "common.cuh"

namespace ds {

struct ReduceArgs {
    uint64_t in;        // n values, raw bits: u16 for fp16/bf16, u32 for fp32
    uint64_t partials;  // >= g partial bit patterns (u32 each)
    uint64_t out;       // u32: result bits
    uint64_t ticket;    // u32 counter, 0 at launch; reset by the last block
    int64_t n;
    int32_t fmt;        // 0 fp16, 1 bf16, 2 fp32 (FloatFormatKind order)
    int32_t combine;    // 1: last block folds partials (full reduction_result)
};

__device__ __forceinline__ uint32_t add_rn(int fmt, uint32_t a, uint32_t b) {
    if (fmt == 0) {
        uint16_t r;
        asm("add.rn.f16 %0, %1, %2;" : "=h"(r) : "h"((uint16_t)a), "h"((uint16_t)b));
        return r;
    } else if (fmt == 1) {
        uint16_t r;
        asm("add.rn.bf16 %0, %1, %2;" : "=h"(r) : "h"((uint16_t)a), "h"((uint16_t)b));
        return r;
    } else {
        float r;
        asm("add.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(__uint_as_float(a)), "f"(__uint_as_float(b)));
        return __float_as_uint(r);
    }
}

__device__ __forceinline__ uint32_t load_val(int fmt, const void* base, int64_t i) {
    if (fmt == 2) return reinterpret_cast<const uint32_t*>(base)[i];
    return reinterpret_cast<const uint16_t*>(base)[i];
}

// smem staging of up to kChunk values; thread 0 folds sequentially
__device__ void body_reduce(const BodyCtx& c) {
    const ReduceArgs& a = *reinterpret_cast<const ReduceArgs*>(c.args);
    const uint32_t g = c.gx * c.gy * c.gz;
    const uint32_t blk = c.bx + c.gx * (c.by + c.gy * c.bz);
    const int64_t lo = (int64_t)blk * a.n / g;
    const int64_t hi = (int64_t)(blk + 1) * a.n / g;
    uint32_t* stage = reinterpret_cast<uint32_t*>(c.smem);
    const int64_t kChunk = 16384;
    uint32_t acc = 0;  // FloatValue::finite(0) for an empty chunk (+0 bits)
    bool first = true;
    const void* in = reinterpret_cast<const void*>(a.in);
    for (int64_t base = lo; base < hi; base += kChunk) {
        int64_t cnt = hi - base < kChunk ? hi - base : kChunk;
        for (int64_t i = ltid(); i < cnt; i += kBodyThreads) stage[i] = load_val(a.fmt, in, base + i);
        body_sync();
        if (ltid() == 0) {
            int64_t i = 0;
            if (first) { acc = stage[0]; i = 1; first = false; }
            for (; i < cnt; ++i) acc = add_rn(a.fmt, acc, stage[i]);
        }
        body_sync();
    }
    __shared__ int is_last_l[2];
    int& is_last = is_last_l[body_lane()];
    if (ltid() == 0) {
        uint32_t* partials = reinterpret_cast<uint32_t*>(a.partials);
        partials[blk] = acc;
        is_last = 0;
        if (a.combine) {
            __threadfence();
            uint32_t t = atomicAdd(reinterpret_cast<uint32_t*>(a.ticket), 1u);
            is_last = (t == g - 1);
        }
    }
    body_sync();
    if (is_last && ltid() == 0) {
        __threadfence();
        const volatile uint32_t* p = reinterpret_cast<const volatile uint32_t*>(a.partials);
        uint32_t r = p[0];
        for (uint32_t i = 1; i < g; ++i) r = add_rn(a.fmt, r, p[i]);
        *reinterpret_cast<uint32_t*>(a.out) = r;
        *reinterpret_cast<uint32_t*>(a.ticket) = 0;  // ready for the next launch
    }
    body_sync();
}

// ---------------------------------------------------------------------------
// Output checksum (parity evidence at full size): launch seq's block b writes
// partial[(seq % cap) * grid + b] = sum over its words w_i of w_i * (2i + 1)
// mod 2^64 (i = global 32-bit word index).  Integer arithmetic: the value
// depends only on the buffer's bits, never on scheduling, and the per-launch
// slot lets the host check every launch of a long co-located run against a
// plain-grid solo run (solo: seq = 0).
// ---------------------------------------------------------------------------
struct ChecksumArgs {
    uint64_t src;       // buffer (32-bit words)
    uint64_t partials;  // u64 [cap][grid]
    int64_t n_words;
    int32_t cap;
    int32_t pad;
};

__device__ void body_checksum(const BodyCtx& c) {
    const ChecksumArgs& a = *reinterpret_cast<const ChecksumArgs*>(c.args);
    const uint32_t g = c.gx * c.gy * c.gz;
    const uint32_t blk = c.bx + c.gx * (c.by + c.gy * c.bz);
    const int64_t lo = (int64_t)blk * a.n_words / g;
    const int64_t hi = (int64_t)(blk + 1) * a.n_words / g;
    const uint32_t* w = reinterpret_cast<const uint32_t*>(a.src);
    unsigned long long h = 0;
    // 16-B loads on the aligned interior, scalar head / tail
    const int64_t lo4 = (lo + 3) & ~3ll, hi4 = hi & ~3ll;
    if (lo4 < hi4) {
        for (int64_t i = lo4 + 4 * (int64_t)ltid(); i < hi4; i += 4 * kBodyThreads) {
            const uint4 v = __ldcs(reinterpret_cast<const uint4*>(w + i));
            const unsigned long long m = 2ull * (unsigned long long)i + 1ull;
            h += (unsigned long long)v.x * m + (unsigned long long)v.y * (m + 2) + (unsigned long long)v.z * (m + 4) +
                 (unsigned long long)v.w * (m + 6);
        }
        for (int64_t i = lo + ltid(); i < lo4; i += kBodyThreads) h += (unsigned long long)w[i] * (2ull * i + 1ull);
        for (int64_t i = hi4 + ltid(); i < hi; i += kBodyThreads) h += (unsigned long long)w[i] * (2ull * i + 1ull);
    } else {
        for (int64_t i = lo + ltid(); i < hi; i += kBodyThreads) h += (unsigned long long)w[i] * (2ull * i + 1ull);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    __shared__ unsigned long long red_l[2][8];
    unsigned long long* red = red_l[body_lane()];
    if ((ltid() & 31) == 0) red[ltid() >> 5] = h;
    body_sync();
    if (ltid() == 0) {
        unsigned long long t = 0;
        for (int i = 0; i < kBodyThreads / 32; ++i) t += red[i];
        const uint32_t slot = a.cap > 0 ? c.seq % (uint32_t)a.cap : 0u;
        reinterpret_cast<unsigned long long*>(a.partials)[(size_t)slot * g + blk] = t;
    }
    body_sync();
}

}  // namespace ds
