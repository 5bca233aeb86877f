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
    uint64_t dbg;       // optional phase timestamps [grid][8] (0 = off)
    uint64_t w_packed;  // W pre-packed as SWIZZLE_128B [N/128][K/64][128][64] tiles (0 = use tmW)
};

constexpr int kGemvBN = 32;
constexpr int kGemvStages = kCtasPerSm == 2 ? 5 : 8;
// epilogue scratch [128][33] fp32 + rvec/flag reuses the TMA ring: every
// stage has been consumed once the accumulator is complete
constexpr uint32_t kGemvScratch = 0;

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
    uint64_t* dbg = a.dbg ? reinterpret_cast<uint64_t*>(a.dbg) + (size_t)t * 8 : nullptr;
    if (dbg && ltid() == 0) dbg[0] = globaltimer();
    tc_mainloop<kGemvBN, kGemvStages>(base, &a.tmW, &a.tmX, n_blk * kTcBM, 0, kb0, kb1, c.tmem_base, true,
                                      reinterpret_cast<const char*>(a.w_packed), KB);
    if (dbg && ltid() == 128) dbg[1] = globaltimer();
    const int warp = ltid() >> 5, lane = ltid() & 31;
    float* scratch = reinterpret_cast<float*>(base + kGemvScratch);  // [128][33] + rvec[32] + flag
    float* rvec = scratch + 128 * 33;
    volatile int* flag = reinterpret_cast<volatile int*>(scratch + 128 * 33 + 32 + 16);
    const int q = warp & 3;
    const int row = q * 32 + lane;  // epilogue warps: row within the slab
    const int n = n_blk * kTcBM + row;
    float v[32];
    if (warp >= 4) {
        uint32_t raw[32];
        tc::tmem_ld_32x32b_x32(c.tmem_base + ((uint32_t)(q * 32) << 16), raw);
        tc::tmem_ld_wait();
#pragma unroll
        for (int b = 0; b < 32; ++b) v[b] = __uint_as_float(raw[b]);
    }
    bool proceed = true;
    if (a.S > 1) {
        if (warp >= 4) {
            float4* w = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.ws) + ((size_t)s * a.N + n) * 32);
#pragma unroll
            for (int j = 0; j < 8; ++j) w[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
        body_sync();
        if (ltid() == 0) {
            // one release/acquire RMW publishes the whole CTA's partial (the
            // bar.sync above orders the other threads' stores before it)
            uint32_t tk;
            asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;"
                         : "=r"(tk) : "l"(reinterpret_cast<uint32_t*>(a.counters) + n_blk) : "memory");
            *flag = (tk == (uint32_t)a.S - 1);
        }
        body_sync();
        proceed = *flag != 0;
        if (dbg && ltid() == 0) dbg[2] = globaltimer() | ((uint64_t)proceed << 63);
        if (proceed) {
            // all 256 threads, coalesced: thread owns float4 f = ltid() + 256 j
            // of the slab's [128 rows][32] block; partials summed in the fixed
            // order s = 0..S-1
            __threadfence();
            const float4* wsb = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(a.ws) +
                                                                (size_t)n_blk * kTcBM * 32);
            const size_t sstride4 = (size_t)a.N * 8;
            float4 acc[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 3
            for (int sp = 0; sp < a.S; ++sp) {
                float4 x[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) x[j] = __ldcg(wsb + sp * sstride4 + ltid() + 256 * j);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    acc[j].x += x[j].x;
                    acc[j].y += x[j].y;
                    acc[j].z += x[j].z;
                    acc[j].w += x[j].w;
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int f = ltid() + 256 * j;
                float* dst = scratch + (f >> 3) * 33 + (f & 7) * 4;
                dst[0] = acc[j].x;
                dst[1] = acc[j].y;
                dst[2] = acc[j].z;
                dst[3] = acc[j].w;
            }
            if (ltid() == 0) reinterpret_cast<uint32_t*>(a.counters)[n_blk] = 0;
            body_sync();
            if (warp >= 4) {
#pragma unroll
                for (int b = 0; b < 32; ++b) v[b] = scratch[row * 33 + b];
            }
            body_sync();  // scratch rows are rewritten by the mode epilogues below
            if (dbg && ltid() == 0) dbg[3] = globaltimer();
        }
    }
    if (warp >= 4) {
        if (proceed) {
            // RMSNorm of the input rows folded in as a per-row scale
            if (a.stats_in) {
                float* red = scratch + 128 * 33 + 64;  // [4][32]
                {
                    const float* st = reinterpret_cast<const float*>(a.stats_in);
                    const int p0 = q * a.P_in / 4, p1 = (q + 1) * a.P_in / 4;
                    float ss = 0.f;
#pragma unroll 8
                    for (int p = p0; p < p1; ++p) ss += __ldcg(st + p * 32 + lane);
                    red[q * 32 + lane] = ss;
                }
                epi_sync();
                if (warp == 4) {
                    const float ss = ((red[lane] + red[32 + lane]) + red[64 + lane]) + red[96 + lane];
                    rvec[lane] = rsqrtf(ss / (float)a.K + a.eps);
                }
                epi_sync();
#pragma unroll
                for (int b = 0; b < 32; ++b) v[b] *= rvec[b];
            }
            if (dbg && ltid() == 128) dbg[4] = globaltimer();
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
                {  // fixed-order sum over the 128 rows: 4 quarter sums, then in order
                    float* red = scratch + 128 * 33 + 64;
                    float ss = 0.f;
#pragma unroll 8
                    for (int r = q * 32; r < q * 32 + 32; ++r) ss += scratch[r * 33 + lane];
                    red[q * 32 + lane] = ss;
                    epi_sync();
                    if (warp == 4)
                        reinterpret_cast<float*>(a.stats_out)[n_blk * 32 + lane] =
                            ((red[lane] + red[32 + lane]) + red[64 + lane]) + red[96 + lane];
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
    if (dbg && ltid() == 128) dbg[5] = globaltimer();
    tc_teardown<kGemvBN, kGemvStages>(base);
    if (dbg && ltid() == 0) dbg[6] = globaltimer();
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

constexpr int kAttnChunk = 32;   // KV positions per staged chunk (8 KB of K + 8 KB of V)
constexpr int kAttnStages = 4;
constexpr uint32_t kAttnStageBytes = 2 * kAttnChunk * 128 * 2;
constexpr uint32_t kAttnBarOff = kAttnStages * kAttnStageBytes;       // 64 KB
constexpr uint32_t kAttnMergeOff = kAttnBarOff + 1024;               // [8][4][130] fp32
constexpr uint32_t kAttnSmem = kAttnMergeOff + 8 * 4 * 130 * 4 + 1024;

__device__ void body_attn_decode(const BodyCtx& c) {
    const AttnArgs& a = *reinterpret_cast<const AttnArgs*>(c.args);
    const int t = c.bx + c.gx * (c.by + c.gy * c.bz);
    const int bh = t % 256, sp = t / 256;
    const int b = bh >> 3, h = bh & 7;
    const int warp = ltid() >> 5, lane = ltid() & 31;
    const int p0 = (int)((int64_t)sp * a.L / a.S), p1 = (int)((int64_t)(sp + 1) * a.L / a.S);
    const int nch = (p1 - p0 + kAttnChunk - 1) / kAttnChunk;
    char* base = align1024(c.smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(base + kAttnBarOff);
    uint64_t* empty = full + kAttnStages;
    const uint16_t* kb = reinterpret_cast<const uint16_t*>(a.kcache) + ((size_t)(b * 8 + h) * a.Lmax) * 128;
    const uint16_t* vb = reinterpret_cast<const uint16_t*>(a.vcache) + ((size_t)(b * 8 + h) * a.Lmax) * 128;
    // the KV stream is read once per step: TMA bulk copies into a 4-deep smem ring
    auto issue = [&](int i) {
        const int s = i % kAttnStages;
        const int r0 = p0 + i * kAttnChunk;
        const int rows = min(kAttnChunk, p1 - r0);
        const uint32_t bytes = rows * 256;
        char* dst = base + s * kAttnStageBytes;
        const uint64_t pol = tc::policy_evict_first();
        tc::mbar_arrive_expect_tx(&full[s], 2 * bytes);
        tc::bulk_g2s_hint(dst, kb + (size_t)r0 * 128, bytes, &full[s], pol);
        tc::bulk_g2s_hint(dst + kAttnChunk * 256, vb + (size_t)r0 * 128, bytes, &full[s], pol);
    };
    if (ltid() == 0) {
        for (int s = 0; s < kAttnStages; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 8);
        }
        tc::fence_mbar_init();
        for (int i = 0; i < min(kAttnStages, nch); ++i) issue(i);
    }
    body_sync();
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
    float m[4], l[4], acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        m[i] = kNegInf;
        l[i] = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    }
    for (int ci = 0; ci < nch; ++ci) {
        const int s = ci % kAttnStages;
        const uint32_t ph = (ci / kAttnStages) & 1;
        tc::mbar_wait(&full[s], ph);
        const char* stg = base + s * kAttnStageBytes;
        const int r0 = p0 + ci * kAttnChunk;
        const int rows = min(kAttnChunk, p1 - r0);
#pragma unroll
        for (int u = 0; u < kAttnChunk / 8; ++u) {
            const int r = warp * (kAttnChunk / 8) + u;
            if (r >= rows) break;
            const uint2 kr = *reinterpret_cast<const uint2*>(stg + r * 256 + lane * 8);
            const uint2 vr = *reinterpret_cast<const uint2*>(stg + kAttnChunk * 256 + r * 256 + lane * 8);
            float kf[4] = {__uint_as_float(kr.x << 16), __uint_as_float(kr.x & 0xffff0000u),
                           __uint_as_float(kr.y << 16), __uint_as_float(kr.y & 0xffff0000u)};
            float vf[4] = {__uint_as_float(vr.x << 16), __uint_as_float(vr.x & 0xffff0000u),
                           __uint_as_float(vr.y << 16), __uint_as_float(vr.y & 0xffff0000u)};
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
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&empty[s]);
        if (ltid() == 0 && ci + kAttnStages < nch) {
            tc::mbar_wait(&empty[s], ph);  // all 8 warps released this slot
            issue(ci + kAttnStages);
        }
    }
    // merge the 8 warps in order (smem: [8][4][130])
    float* sm = reinterpret_cast<float*>(base + kAttnMergeOff);
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
    if (ltid() == 0)
        for (int s = 0; s < 2 * kAttnStages; ++s) tc::mbar_inval(&full[s]);
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
// on ties.  Logical block t -> (row b = t % 32, chunk c = t / 32); each chunk
// writes (max, idx); the row's last chunk (ticket) reduces chunks 0..C-1 in
// order.  Deterministic under any schedule.
// ---------------------------------------------------------------------------
struct ArgmaxArgs {
    uint64_t logits;    // bf16 [32][vocab]
    uint64_t tokens;    // int32 [32]
    uint64_t ws;        // {float, int} [32][chunks]
    uint64_t counters;  // u32 [32]
    int32_t vocab;
    int32_t chunks;
};

__device__ __forceinline__ void amax_merge(float& f, int& i, float f2, int i2) {
    if (f2 > f || (f2 == f && i2 < i)) {
        f = f2;
        i = i2;
    }
}

__device__ void body_argmax(const BodyCtx& c) {
    const ArgmaxArgs& a = *reinterpret_cast<const ArgmaxArgs*>(c.args);
    const int t = c.bx + c.gx * (c.by + c.gy * c.bz);
    const int b = t % 32, ch = t / 32;
    const int v0 = (int)((int64_t)ch * a.vocab / a.chunks), v1 = (int)((int64_t)(ch + 1) * a.vocab / a.chunks);
    const uint16_t* row = reinterpret_cast<const uint16_t*>(a.logits) + (size_t)b * a.vocab;
    float best = kNegInf;
    int idx = 0x7fffffff;
    // 16-B vector body over the 8-aligned interior, scalar edges
    const int va = (v0 + 7) & ~7, vb = v1 & ~7;
    for (int v = v0 + (int)ltid(); v < min(va, v1); v += kBodyThreads) amax_merge(best, idx, bf16_to_f(row[v]), v);
    for (int v = va + 8 * (int)ltid(); v < vb; v += 8 * kBodyThreads) {
        uint4 q = __ldcs(reinterpret_cast<const uint4*>(row + v));
        uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            amax_merge(best, idx, __uint_as_float(w[j] << 16), v + 2 * j);
            amax_merge(best, idx, __uint_as_float(w[j] & 0xffff0000u), v + 2 * j + 1);
        }
    }
    for (int v = max(vb, va) + (int)ltid(); v < v1; v += kBodyThreads) amax_merge(best, idx, bf16_to_f(row[v]), v);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        float f2 = __shfl_xor_sync(0xffffffffu, best, o);
        int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
        amax_merge(best, idx, f2, i2);
    }
    __shared__ float sb_l[2][8];
    __shared__ int si_l[2][8];
    __shared__ int last_l[2];
    float* sb = sb_l[body_lane()];
    int* si = si_l[body_lane()];
    const int warp = ltid() >> 5, lane = ltid() & 31;
    if (lane == 0) {
        sb[warp] = best;
        si[warp] = idx;
    }
    body_sync();
    if (ltid() == 0) {
        float f = sb[0];
        int i = si[0];
        for (int w = 1; w < 8; ++w) amax_merge(f, i, sb[w], si[w]);
        float* ws = reinterpret_cast<float*>(a.ws) + ((size_t)b * a.chunks + ch) * 2;
        ws[0] = f;
        reinterpret_cast<int*>(ws)[1] = i;
        __threadfence();
        uint32_t tk = atomicAdd(reinterpret_cast<uint32_t*>(a.counters) + b, 1u);
        last_l[body_lane()] = tk == (uint32_t)a.chunks - 1;
        if (tk == (uint32_t)a.chunks - 1) {
            __threadfence();
            const float* wr = reinterpret_cast<const float*>(a.ws) + (size_t)b * a.chunks * 2;
            float bf = __ldcg(wr);
            int bi = __ldcg(reinterpret_cast<const int*>(wr) + 1);
            for (int k = 1; k < a.chunks; ++k)
                amax_merge(bf, bi, __ldcg(wr + 2 * k), __ldcg(reinterpret_cast<const int*>(wr + 2 * k) + 1));
            reinterpret_cast<int*>(a.tokens)[b] = bi;
            reinterpret_cast<uint32_t*>(a.counters)[b] = 0;
        }
    }
    body_sync();
}

}  // namespace ds
