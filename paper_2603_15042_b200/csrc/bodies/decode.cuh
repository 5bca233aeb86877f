// Decode tenant (Llama-3-8B-shaped, batch 32): projection GEMV on tcgen05,
// GQA decode attention, and the RMS statistics that let RMSNorm fold into the
// projections' epilogues.  All are HBM-bound; all reductions run in a fixed
// order that depends only on the logical block index, so a decode step's
// outputs are bit-identical solo or as a coroutine under any SM quota.
#pragma once
#include "common.cuh"
#include "gemm_tc.cuh"

namespace ds {

#define kNegInf (-__int_as_float(0x7f800000))

// ---------------------------------------------------------------------------
// Projection: y[b][n] = sum_k W[n][k] x[b][k]  (b < 32), swap-AB on tcgen05:
// D[128 weight rows][32 batch] with the weight slab as the M operand.
// Logical block t -> (row slab n_blk = t % nb, K-split s = t / nb).  With
// S > 1 each block writes fp32 partials and the block that retires last for
// its slab (ticket) sums s = 0..S-1 in order and runs the epilogue.
// ---------------------------------------------------------------------------
enum GemvMode : int32_t { kGemvStore = 0, kGemvResid = 1, kGemvSiluMul = 2, kGemvQKV = 3 };

struct GemvArgs {
    TmaDesc tmW;        // W [N][K] bf16, box {64, 128}
    TmaDesc tmX;        // X [32][K] bf16, box {64, 32}
    uint64_t out;       // bf16 output (layout by mode)
    uint64_t resid;     // bf16 [32][N] residual (kGemvResid)
    uint64_t ws;        // fp32 [S][N][32] split-K partials
    uint64_t counters;  // u32 [N/128] split-K tickets (0 at rest)
    uint64_t stats_in;  // fp32 [P_in][32] sum of squares of X rows (RMSNorm), 0 = none
    uint64_t stats_out; // fp32 [N/128][32] sum of squares of the output rows (kGemvResid)
    uint64_t kcache;    // kGemvQKV: bf16 [32][8][Lmax][128] for this layer
    uint64_t vcache;
    int32_t N, K, S, mode;
    int32_t P_in;
    float eps;
    int32_t pos;        // kGemvQKV: cache row written this step
    int32_t Lmax;
    int32_t q_dim, kv_dim;
    int32_t pad0, pad1;
};

constexpr int kGemvBN = 32;
constexpr int kGemvStages = kCtasPerSm == 2 ? 4 : 8;
constexpr uint32_t kGemvScratch = TcSmem<kGemvBN, kGemvStages>::kBytes;  // epilogue scratch offset

__device__ __forceinline__ float bf16_to_f(uint16_t v) { return __uint_as_float((uint32_t)v << 16); }
__device__ __forceinline__ uint16_t f_to_bf16(float f) {
    __nv_bfloat16 h = __float2bfloat16_rn(f);
    return *reinterpret_cast<uint16_t*>(&h);
}


__device__ void body_gemv_bf16(const BodyCtx& c) {
    const GemvArgs& a = *reinterpret_cast<const GemvArgs*>(c.args);
    char* base = align1024(c.smem);
    const int nb = a.N / kTcBM;
    const int t = c.bx + c.gx * (c.by + c.gy * c.bz);
    const int n_blk = t % nb, s = t / nb;
    const int KB = a.K / kTcBK;
    const int kb0 = (int)((int64_t)s * KB / a.S), kb1 = (int)((int64_t)(s + 1) * KB / a.S);
    tc_mainloop<kGemvBN, kGemvStages>(base, &a.tmW, &a.tmX, n_blk * kTcBM, 0, kb0, kb1, c.tmem_base, true);
    const int warp = ltid() >> 5, lane = ltid() & 31;
    if (warp >= 4) {
        const int q = warp & 3;
        const int row = q * 32 + lane;  // row within the slab
        const int n = n_blk * kTcBM + row;
        float* scratch = reinterpret_cast<float*>(base + kGemvScratch);  // [128][33] + flags
        volatile int* flag = reinterpret_cast<volatile int*>(scratch + 128 * 33 + 32);
        float* rvec = scratch + 128 * 33;
        uint32_t raw[32];
        tc::tmem_ld_32x32b_x32(c.tmem_base + ((uint32_t)(q * 32) << 16), raw);
        tc::tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int b = 0; b < 32; ++b) v[b] = __uint_as_float(raw[b]);
        bool proceed = true;
        if (a.S > 1) {
            float4* w = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.ws) + ((size_t)s * a.N + n) * 32);
#pragma unroll
            for (int j = 0; j < 8; ++j) w[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            __threadfence();
            epi_sync();
            if (warp == 4 && lane == 0) {
                uint32_t tk = atomicAdd(reinterpret_cast<uint32_t*>(a.counters) + n_blk, 1u);
                *flag = (tk == (uint32_t)a.S - 1);
            }
            epi_sync();
            proceed = *flag != 0;
            if (proceed) {
                __threadfence();
                const float* wsr = reinterpret_cast<const float*>(a.ws);
#pragma unroll
                for (int b = 0; b < 32; ++b) v[b] = 0.f;
                for (int sp = 0; sp < a.S; ++sp) {  // fixed order
                    const float4* p = reinterpret_cast<const float4*>(wsr + ((size_t)sp * a.N + n) * 32);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        float4 x = __ldcg(p + j);
                        v[4 * j] += x.x;
                        v[4 * j + 1] += x.y;
                        v[4 * j + 2] += x.z;
                        v[4 * j + 3] += x.w;
                    }
                }
                if (warp == 4 && lane == 0) reinterpret_cast<uint32_t*>(a.counters)[n_blk] = 0;
            }
        }
        if (proceed) {
            // RMSNorm of the input rows folded in as a per-row scale
            if (a.stats_in) {
                if (warp == 4) {
                    const float* st = reinterpret_cast<const float*>(a.stats_in);
                    float ss = 0.f;
                    for (int p = 0; p < a.P_in; ++p) ss += __ldcg(st + p * 32 + lane);
                    rvec[lane] = rsqrtf(ss / (float)a.K + a.eps);
                }
                epi_sync();
#pragma unroll
                for (int b = 0; b < 32; ++b) v[b] *= rvec[b];
            }
            if (a.mode == kGemvStore) {
                uint16_t* out = reinterpret_cast<uint16_t*>(a.out);
#pragma unroll
                for (int b = 0; b < 32; ++b) out[(size_t)b * a.N + n] = f_to_bf16(v[b]);
            } else if (a.mode == kGemvResid) {
                const uint16_t* res = reinterpret_cast<const uint16_t*>(a.resid);
                uint16_t* out = reinterpret_cast<uint16_t*>(a.out);
#pragma unroll
                for (int b = 0; b < 32; ++b) {
                    float h = bf16_to_f(__ldcg(res + (size_t)b * a.N + n)) + v[b];
                    uint16_t hb = f_to_bf16(h);
                    out[(size_t)b * a.N + n] = hb;
                    float hr = bf16_to_f(hb);
                    scratch[row * 33 + b] = hr * hr;
                }
                epi_sync();
                if (warp == 4) {  // lane = b: fixed-order sum over the 128 rows
                    float ss = 0.f;
                    for (int r = 0; r < 128; ++r) ss += scratch[r * 33 + lane];
                    reinterpret_cast<float*>(a.stats_out)[n_blk * 32 + lane] = ss;
                }
            } else if (a.mode == kGemvSiluMul) {
                // slab rows [0,64) are gate features, [64,128) the matching up features
#pragma unroll
                for (int b = 0; b < 32; ++b) scratch[row * 33 + b] = v[b];
                epi_sync();
                if (row < 64) {
                    uint16_t* out = reinterpret_cast<uint16_t*>(a.out);
                    const int f = n_blk * 64 + row;
                    const int F = a.N / 2;
#pragma unroll
                    for (int b = 0; b < 32; ++b) {
                        float g = scratch[row * 33 + b], u = scratch[(row + 64) * 33 + b];
                        float act = g / (1.f + __expf(-g)) * u;
                        out[(size_t)b * F + f] = f_to_bf16(act);
                    }
                }
            } else if (a.mode == kGemvQKV) {
                if (n < a.q_dim) {
                    uint16_t* out = reinterpret_cast<uint16_t*>(a.out);
#pragma unroll
                    for (int b = 0; b < 32; ++b) out[(size_t)b * a.q_dim + n] = f_to_bf16(v[b]);
                } else {
                    const bool is_k = n < a.q_dim + a.kv_dim;
                    const int m = n - a.q_dim - (is_k ? 0 : a.kv_dim);
                    const int h = m >> 7, d = m & 127;
                    const int nkv = a.kv_dim >> 7;
                    uint16_t* cache = reinterpret_cast<uint16_t*>(is_k ? a.kcache : a.vcache);
#pragma unroll
                    for (int b = 0; b < 32; ++b)
                        cache[(((size_t)b * nkv + h) * a.Lmax + a.pos) * 128 + d] = f_to_bf16(v[b]);
                }
            }
        }
    }
    tc_teardown<kGemvBN, kGemvStages>(base);
}

// ---------------------------------------------------------------------------
// RMS statistics of the decode input rows: stats[0][b] = sum_k x[b][k]^2,
// fixed-order (lane-strided partials, fixed shuffle tree).  grid 1.
// ---------------------------------------------------------------------------
struct RmsArgs {
    uint64_t x;      // bf16 [32][K]
    uint64_t stats;  // fp32 [1][32]
    int32_t K;
    int32_t pad;
};

__device__ void body_rmsnorm(const BodyCtx& c) {
    // grid 32: block b reduces row b in a fixed order (16-B loads, fixed tree)
    const RmsArgs& a = *reinterpret_cast<const RmsArgs*>(c.args);
    const int b = c.bx, warp = ltid() >> 5, lane = ltid() & 31;
    const uint4* x = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.x) + (size_t)b * a.K);
    float ss = 0.f;
    for (int i = ltid(); i < a.K / 8; i += kBodyThreads) {
        uint4 v = __ldcg(x + i);
        uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float lo = __uint_as_float(w[j] << 16), hi = __uint_as_float(w[j] & 0xffff0000u);
            ss += lo * lo + hi * hi;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    __shared__ float part_l[2][8];
    float* part = part_l[body_lane()];
    if (lane == 0) part[warp] = ss;
    body_sync();
    if (ltid() == 0) {
        float t = 0.f;
        for (int w = 0; w < 8; ++w) t += part[w];
        reinterpret_cast<float*>(a.stats)[b] = t;
    }
    body_sync();
}

// ---------------------------------------------------------------------------
// GQA decode attention (32 q heads, 8 kv heads, d = 128, batch 32) over a
// KV cache of L positions.  Logical block t -> (b, kv head h, split sp).
// 8 warps stride over the split's positions with an online softmax per warp;
// warps merge in order 0..7, splits merge in order 0..S-1 (last block).
// ---------------------------------------------------------------------------
struct AttnArgs {
    uint64_t q;         // bf16 [32][32*128]
    uint64_t kcache;    // bf16 [32][8][Lmax][128]
    uint64_t vcache;
    uint64_t out;       // bf16 [32][32*128]
    uint64_t ws;        // fp32 [256][S][4][130]
    uint64_t counters;  // u32 [256]
    int32_t L, Lmax, S;
    float scale;        // 1/sqrt(128)
};

__device__ void body_attn_decode(const BodyCtx& c) {
    const AttnArgs& a = *reinterpret_cast<const AttnArgs*>(c.args);
    const int t = c.bx + c.gx * (c.by + c.gy * c.bz);
    const int bh = t % 256, sp = t / 256;
    const int b = bh >> 3, h = bh & 7;
    const int warp = ltid() >> 5, lane = ltid() & 31;
    const int p0 = (int)((int64_t)sp * a.L / a.S), p1 = (int)((int64_t)(sp + 1) * a.L / a.S);
    const uint16_t* qb = reinterpret_cast<const uint16_t*>(a.q) + (size_t)b * 4096 + (h * 4) * 128;
    float qv[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        uint2 raw = __ldcg(reinterpret_cast<const uint2*>(qb + i * 128 + lane * 4));
        qv[i][0] = __uint_as_float(raw.x << 16) * a.scale;
        qv[i][1] = __uint_as_float(raw.x & 0xffff0000u) * a.scale;
        qv[i][2] = __uint_as_float(raw.y << 16) * a.scale;
        qv[i][3] = __uint_as_float(raw.y & 0xffff0000u) * a.scale;
    }
    const uint16_t* kb = reinterpret_cast<const uint16_t*>(a.kcache) + ((size_t)(b * 8 + h) * a.Lmax) * 128;
    const uint16_t* vb = reinterpret_cast<const uint16_t*>(a.vcache) + ((size_t)(b * 8 + h) * a.Lmax) * 128;
    float m[4], l[4], acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        m[i] = kNegInf;
        l[i] = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    }
    constexpr int U = 8;
    for (int pbase = p0 + warp * U; pbase < p1; pbase += 8 * U) {
        uint2 kr[U], vr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int p = pbase + u;
            if (p < p1) {
                kr[u] = __ldcs(reinterpret_cast<const uint2*>(kb + (size_t)p * 128 + lane * 4));
                vr[u] = __ldcs(reinterpret_cast<const uint2*>(vb + (size_t)p * 128 + lane * 4));
            } else {
                kr[u] = make_uint2(0, 0);
                vr[u] = make_uint2(0, 0);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int p = pbase + u;
            if (p >= p1) break;
            float kf[4] = {__uint_as_float(kr[u].x << 16), __uint_as_float(kr[u].x & 0xffff0000u),
                           __uint_as_float(kr[u].y << 16), __uint_as_float(kr[u].y & 0xffff0000u)};
            float vf[4] = {__uint_as_float(vr[u].x << 16), __uint_as_float(vr[u].x & 0xffff0000u),
                           __uint_as_float(vr[u].y << 16), __uint_as_float(vr[u].y & 0xffff0000u)};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                float d = qv[i][0] * kf[0] + qv[i][1] * kf[1] + qv[i][2] * kf[2] + qv[i][3] * kf[3];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
                const float mn = fmaxf(m[i], d);
                const float alpha = __expf(m[i] - mn);
                const float pexp = __expf(d - mn);
                l[i] = l[i] * alpha + pexp;
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = acc[i][j] * alpha + pexp * vf[j];
                m[i] = mn;
            }
        }
    }
    // merge the 8 warps in order (smem: [8][4][130])
    float* sm = reinterpret_cast<float*>(c.smem);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float* w = sm + (warp * 4 + i) * 130;
#pragma unroll
        for (int j = 0; j < 4; ++j) w[lane * 4 + j] = acc[i][j];
        if (lane == 0) {
            w[128] = m[i];
            w[129] = l[i];
        }
    }
    body_sync();
    // thread -> (head i = tid / 64, dims 2*(tid%64), +1)
    const int i = ltid() >> 6, d0 = (ltid() & 63) * 2;
    float M = kNegInf;
    for (int w = 0; w < 8; ++w) M = fmaxf(M, sm[(w * 4 + i) * 130 + 128]);
    float Ls = 0.f, A0 = 0.f, A1 = 0.f;
    for (int w = 0; w < 8; ++w) {
        const float* src = sm + (w * 4 + i) * 130;
        const float mw = src[128];
        const float f = (mw == kNegInf) ? 0.f : __expf(mw - M);
        Ls += src[129] * f;
        A0 += src[d0] * f;
        A1 += src[d0 + 1] * f;
    }
    bool write_out = true;
    __shared__ int last_flag_l[2];
    int& last_flag = last_flag_l[body_lane()];
    if (a.S > 1) {
        float* ws = reinterpret_cast<float*>(a.ws) + ((size_t)bh * a.S + sp) * 4 * 130 + i * 130;
        ws[d0] = A0;
        ws[d0 + 1] = A1;
        if ((ltid() & 63) == 0) {
            ws[128] = M;
            ws[129] = Ls;
        }
        __threadfence();
        body_sync();
        if (ltid() == 0) {
            uint32_t tk = atomicAdd(reinterpret_cast<uint32_t*>(a.counters) + bh, 1u);
            last_flag = tk == (uint32_t)a.S - 1;
        }
        body_sync();
        write_out = last_flag != 0;
        if (write_out) {
            __threadfence();
            const float* wsb = reinterpret_cast<const float*>(a.ws) + (size_t)bh * a.S * 4 * 130 + i * 130;
            M = kNegInf;
            for (int s2 = 0; s2 < a.S; ++s2) M = fmaxf(M, __ldcg(wsb + s2 * 4 * 130 + 128));
            Ls = 0.f;
            A0 = 0.f;
            A1 = 0.f;
            for (int s2 = 0; s2 < a.S; ++s2) {
                const float* src = wsb + s2 * 4 * 130;
                const float mw = __ldcg(src + 128);
                const float f = (mw == kNegInf) ? 0.f : __expf(mw - M);
                Ls += __ldcg(src + 129) * f;
                A0 += __ldcg(src + d0) * f;
                A1 += __ldcg(src + d0 + 1) * f;
            }
            if (ltid() == 0) reinterpret_cast<uint32_t*>(a.counters)[bh] = 0;
        }
    }
    if (write_out) {
        const float inv = 1.f / Ls;
        uint32_t* out = reinterpret_cast<uint32_t*>(reinterpret_cast<uint16_t*>(a.out) + (size_t)b * 4096 +
                                                    (h * 4 + i) * 128 + d0);
        *out = pack_bf16x2(A0 * inv, A1 * inv);
    }
    body_sync();
}

}  // namespace ds

namespace ds {

// ---------------------------------------------------------------------------
// Token embedding gather (step input): h[b][:] = E[tok[b]][:].  grid 32.
// ---------------------------------------------------------------------------
struct EmbedArgs {
    uint64_t table;   // bf16 [vocab][d]
    uint64_t tokens;  // int32 [32]
    uint64_t h;       // bf16 [32][d]
    int32_t d, vocab;
};

__device__ void body_embed(const BodyCtx& c) {
    const EmbedArgs& a = *reinterpret_cast<const EmbedArgs*>(c.args);
    const int b = c.bx;
    int tok = __ldcg(reinterpret_cast<const int*>(a.tokens) + b);
    tok = tok < 0 ? 0 : (tok >= a.vocab ? a.vocab - 1 : tok);
    const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.table) + (size_t)tok * a.d);
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(a.h) + (size_t)b * a.d);
    for (int i = ltid(); i < a.d / 8; i += kBodyThreads) dst[i] = __ldcs(src + i);
    body_sync();
}

// ---------------------------------------------------------------------------
// Greedy sampling (step result): tok[b] = argmax_v logits[b][v], lowest index
// on ties.  grid 32, fixed-order tree -> deterministic.
// ---------------------------------------------------------------------------
struct ArgmaxArgs {
    uint64_t logits;  // bf16 [32][vocab]
    uint64_t tokens;  // int32 [32]
    int32_t vocab;
    int32_t pad;
};

__device__ void body_argmax(const BodyCtx& c) {
    const ArgmaxArgs& a = *reinterpret_cast<const ArgmaxArgs*>(c.args);
    const int b = c.bx;
    const uint16_t* row = reinterpret_cast<const uint16_t*>(a.logits) + (size_t)b * a.vocab;
    float best = kNegInf;
    int idx = 0x7fffffff;
    for (int v = ltid(); v < a.vocab; v += kBodyThreads) {
        float f = bf16_to_f(__ldcg(row + v));
        if (f > best) { best = f; idx = v; }
    }
    __shared__ float sb_l[2][kBodyThreads];
    __shared__ int si_l[2][kBodyThreads];
    float* sb = sb_l[body_lane()];
    int* si = si_l[body_lane()];
    sb[ltid()] = best;
    si[ltid()] = idx;
    body_sync();
    for (int o = kBodyThreads / 2; o > 0; o >>= 1) {
        if (ltid() < o) {
            float f2 = sb[ltid() + o];
            int i2 = si[ltid() + o];
            if (f2 > sb[ltid()] || (f2 == sb[ltid()] && i2 < si[ltid()])) {
                sb[ltid()] = f2;
                si[ltid()] = i2;
            }
        }
        body_sync();
    }
    if (ltid() == 0) reinterpret_cast<int*>(a.tokens)[b] = si[0];
    body_sync();
}

}  // namespace ds
