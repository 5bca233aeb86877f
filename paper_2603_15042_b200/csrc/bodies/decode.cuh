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
// Logical block t -> (row slab, k-range) pieces: split-K (t -> slab t % nb,
// split t / nb) or stream-K (equal contiguous runs of (slab, k-block) units
// over any grid size).  A slab's last contributor sums the others' fp32
// partials in ascending k order and runs the epilogue.
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
    uint64_t w_packed;  // W pre-packed as SWIZZLE_128B [N/BM][K/64][BM][64] tiles (0 = use tmW)
    int32_t bm;         // slab rows: 128 (0) or 64 (not for kGemvSiluMul)
    int32_t l2_pf_kb;   // early start: KB of this block's weights past the ring prefetched into L2 before
                        // the dependency resolves (0 = ring only)
    int32_t sk;         // 1: stream-K over the logical grid (equal runs of (slab, k-block) units, <= 2 slabs
                        // per block); 0: split-K S with grid nb * S
    int32_t pair;       // P >= 2: P whole 128-row slabs per block (grid ceil(nb / P)), one continuous weight
                        // stream, slab j's epilogue overlapping slab j+1's; kGemvSiluMul (whose weights always
                        // interleave gate/up rows: 2i gate, 2i+1 up of feature i) or kGemvStore
    int32_t pf_ahead;   // D > 0: every ring issue also prefetches the weight tile D k-blocks ahead into L2
                        // (a sliding window: D x 16 KB more in flight per lane than the smem ring holds)
    int32_t pad_pf;
};

// the host builds these records with ctypes mirrors (_abi.py): pinned offsets
static_assert(offsetof(GemvArgs, out) == 256 && offsetof(GemvArgs, N) == 320 && offsetof(GemvArgs, dbg) == 360 &&
                  offsetof(GemvArgs, w_packed) == 368 && offsetof(GemvArgs, bm) == 376 &&
                  offsetof(GemvArgs, sk) == 384 && offsetof(GemvArgs, pair) == 388 &&
                  offsetof(GemvArgs, pf_ahead) == 392,
              "GemvArgs layout (mirrored in _abi.py)");

constexpr int kGemvBN = 32;
constexpr int kGemvStages = kCtasPerSm == 2 ? 5 : 8;     // 20-KB stages (128-row W tile + X)
constexpr int kGemvStages64 = kCtasPerSm == 2 ? 8 : 12;  // 12-KB stages (64-row W tile + X)
// epilogue scratch [128][33] fp32 + rvec/flag reuses the TMA ring: every
// stage has been consumed once the accumulator is complete
constexpr uint32_t kGemvScratch = 0;
constexpr uint32_t kGemvOwnOff = 32768;  // combiner's own partial (16 KB), clear of the scratch
constexpr uint32_t kGemvResOff = 49152;  // kGemvResid owner: the slab's residual inputs [32 b][BM rows] bf16 (8 KB)

__device__ __forceinline__ float bf16_to_f(uint16_t v) { return __uint_as_float((uint32_t)v << 16); }
__device__ __forceinline__ uint16_t f_to_bf16(float f) {
    __nv_bfloat16 h = __float2bfloat16_rn(f);
    return *reinterpret_cast<uint16_t*>(&h);
}


// A logical block's share of one row slab: k-blocks [ka, kb) of slab n; it is
// contributor c of the slab's nc contributors (ascending k), and the owner
// (combiner) when it holds the slab's last k-block.
struct GemvPiece {
    int n, ka, kb, c, nc;
    bool owner;
};

// Stream-K: unit u = n * KB + k (slab-major), block t covers units
// [t U / G, (t+1) U / G); block_of(u) inverts that.
__device__ __forceinline__ int gemv_block_of(int64_t u, int64_t U, int G) {
    return (int)(((u + 1) * G - 1) / U);
}

// Mainloop over a block's pieces (at most 2, consecutive slabs): one smem
// ring across both; piece p accumulates in TMEM columns [32 p, 32 p + 32).
// The weight operand of step i is packed k-block (n*KB + k) -- in stream-K
// order the block's whole weight range is one contiguous run of 16-KB tiles.
template <int BM, int STAGES>
__device__ __forceinline__ void gemv_mainloop(char* base, const GemvArgs& a, const GemvPiece p0, const GemvPiece p1,
                                              int np, uint32_t tmem_base, const BodyCtx& dep, float* rv_out = nullptr) {
    using L = TcSmem<kGemvBN, STAGES, kTcBK, BM>;
    uint64_t* full = reinterpret_cast<uint64_t*>(base + L::kBarOff);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;  // [2]: per piece in pair mode, else [0] for the whole block
    const int warp = ltid() >> 5, lane = ltid() & 31;
    const int KB = a.K / kTcBK;
    const char* a_packed = reinterpret_cast<const char*>(a.w_packed);
    if (ltid() == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(&tmem_full[0], 1);
        tc::mbar_init(&tmem_full[1], 1);
        tc::fence_mbar_init();
    }
    body_sync();
    // pieces as scalars (a dynamically indexed array would live in local memory)
    const int pn0 = p0.n, pka0 = p0.ka, n0 = p0.kb - p0.ka;
    const int pn1 = np > 1 ? p1.n : pn0, pka1 = np > 1 ? p1.ka : 0;
    const int total = n0 + (np > 1 ? p1.kb - p1.ka : 0);
    // step i -> (slab, k-block)
    auto piece_of = [&](int i, int& n, int& k) {
        const bool second = i >= n0;
        n = second ? pn1 : pn0;
        k = second ? pka1 + (i - n0) : pka0 + i;
    };
    if (warp == 0 && lane == 0) {
        if (desc_fence_needed(dep.st ? &a : nullptr)) {
            if (!a_packed) tc::tma_fence_desc(&a.tmW);
            tc::tma_fence_desc(&a.tmX);
        }
        const uint64_t pol = tc::policy_evict_first();
        auto issue_a = [&](int i) {
            int n, k;
            piece_of(i, n, k);
            char* sa = base + (i % STAGES) * L::kStageBytes;
            if (a_packed)
                tc::bulk_g2s_hint(sa, a_packed + ((size_t)n * KB + k) * L::kABytes, L::kABytes, &full[i % STAGES], pol);
            else
                tc::tma_load_2d_hint(sa, &a.tmW, &full[i % STAGES], k * kTcBK, n * BM, pol);
        };
        auto issue_b = [&](int i) {
            int n, k;
            piece_of(i, n, k);
            tc::tma_load_2d(base + (i % STAGES) * L::kStageBytes + L::kABytes, &a.tmX, &full[i % STAGES], k * kTcBK, 0);
        };
        // the weights (immutable) stream while the previous launch finishes;
        // X (its output) only after wait_prev
        const int pre = min(STAGES, total);
        for (int i = 0; i < pre; ++i) {
            tc::mbar_arrive_expect_tx(&full[i], L::kStageBytes);
            issue_a(i);
        }
        if (a_packed && a.l2_pf_kb && total > pre && wait_prev_streamed(dep)) {
            int n, k;
            piece_of(pre, n, k);
            const char* g0 = a_packed + ((size_t)n * KB + k) * L::kABytes;
            const uint32_t tot = min((uint32_t)(total - pre) * L::kABytes, (uint32_t)a.l2_pf_kb << 10);
            for (uint32_t off = 0; off < tot; off += L::kABytes) tc::bulk_prefetch_l2(g0 + off, min(L::kABytes, tot - off));
        }
        // sliding L2 prefetch D tiles ahead of the ring (weights are immutable,
        // so the first window may go out before the dependency resolves)
        const int D = a_packed ? a.pf_ahead : 0;
        auto prefetch = [&](int j) {
            int n, k;
            piece_of(j, n, k);
            tc::bulk_prefetch_l2(a_packed + ((size_t)n * KB + k) * L::kABytes, L::kABytes);
        };
        for (int j = pre; j < min(total, pre + D); ++j) prefetch(j);
        wait_prev(dep);
        if (dep.dbg) dep.dbg[7] = globaltimer();
        for (int i = 0; i < pre; ++i) issue_b(i);
        for (int i = pre; i < total; ++i) {
            const int s = i % STAGES;
            if (D > 0 && i + D < total) prefetch(i + D);
            tc::mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
            tc::mbar_arrive_expect_tx(&full[s], L::kStageBytes);
            issue_a(i);
            issue_b(i);
        }
    } else if (warp == 1 && lane == 0) {
        constexpr uint32_t idesc = tc::idesc_bf16_f32(BM, kGemvBN);
        for (int i = 0; i < total; ++i) {
            const int s = i % STAGES;
            tc::mbar_wait(&full[s], (i / STAGES) & 1);
            tc::tc_fence_after();
            char* sa = base + s * L::kStageBytes;
            const uint64_t ad = tc::smem_desc_k_sw128(sa), bd = tc::smem_desc_k_sw128(sa + L::kABytes);
            const int p = i < n0 ? 0 : 1;
            const bool first = i == 0 || i == n0;
#pragma unroll
            for (int k = 0; k < kTcBK / 16; ++k)
                tc::mma_bf16(tmem_base + 32 * p, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc, !(first && k == 0));
            tc::mma_commit(&empty[s]);
        }
        tc::mma_commit(&tmem_full[0]);
    }
    if (warp >= 4) {
        // rv_out: the epilogue warps, idle while the ring streams, fold the
        // inputs' RMSNorm statistics (an earlier launch's output: acquired by
        // thread 128's own wait_prev) into the per-row scale now, off the
        // critical path; x 1.0 (exact) without statistics
        if (rv_out) {
            float* red = rv_out + 32;  // [4][32] quarter sums
            const int q = warp & 3;
            if (ltid() == 128) wait_prev(dep);
            epi_sync();
            float ss = 0.f;
            if (a.stats_in) {
                const float* st = reinterpret_cast<const float*>(a.stats_in);
                const int pa = q * a.P_in / 4, pb = (q + 1) * a.P_in / 4;
#pragma unroll 8
                for (int p = pa; p < pb; ++p) ss += __ldcg(st + p * 32 + lane);
            }
            red[q * 32 + lane] = ss;
            epi_sync();
            if (warp == 4)
                rv_out[lane] = a.stats_in ? rsqrtf((((red[lane] + red[32 + lane]) + red[64 + lane]) + red[96 + lane]) /
                                                   (float)a.K + a.eps)
                                          : 1.f;
        }
        tc::mbar_wait(tmem_full, 0);
        tc::tc_fence_after();
    }
}

// SiLU(g) * u, the one formula every gate_up epilogue uses (so the one-slab
// and multi-slab records stay bit-identical): g / (1 + e^-g) with the fast
// reciprocal division (2 instructions instead of the IEEE division's
// slow-path sequence; ~2 ulp fp32, far below the bf16 output rounding).
// e^-g = inf (g < ~-88) gives g * 0 = -0: SiLU's limit.
__device__ __forceinline__ float silu_mul(float g, float u) { return __fdividef(g, 1.f + __expf(-g)) * u; }

// Pair mode (gate_up): SiLU(gate) * up of one slab straight from TMEM.
// Interleaved rows: TMEM lane 2i holds gate feature i of the slab, 2i+1 its
// up partner, so the pair meets by one shuffle; the even lane writes batch
// rows 0-15, the odd lane 16-31.  rvec: the inputs' RMSNorm scales.
__device__ __forceinline__ void gemv_silu_pair_epilogue(const BodyCtx& c, const GemvArgs& a, int slab, uint32_t col,
                                                        const float* rvec) {
    const int q = (ltid() >> 5) & 3, lane = ltid() & 31;
    uint32_t raw[32];
    tc::tmem_ld_32x32b_x32(c.tmem_base + ((uint32_t)(q * 32) << 16) + col, raw);
    tc::tmem_ld_wait();
    const bool odd = lane & 1;
    float mine[16], other[16];
#pragma unroll
    for (int b = 0; b < 16; ++b) {
        // even lane keeps its b < 16 and sends b >= 16; odd lane the reverse
        const float keep = __uint_as_float(raw[odd ? b + 16 : b]);
        const float send = __uint_as_float(raw[odd ? b : b + 16]);
        other[b] = __shfl_xor_sync(0xffffffffu, send, 1);
        mine[b] = keep;
    }
    uint16_t* out = reinterpret_cast<uint16_t*>(a.out);
    const int F = a.N / 2;
    const int f = slab * 64 + q * 16 + (lane >> 1);
    const int b0 = odd ? 16 : 0;
#pragma unroll
    for (int b = 0; b < 16; ++b) {
        const float g = (odd ? other[b] : mine[b]) * rvec[b0 + b];
        const float u = (odd ? mine[b] : other[b]) * rvec[b0 + b];
        out[(size_t)(b0 + b) * F + f] = f_to_bf16(silu_mul(g, u));
    }
}

// Multi-slab blocks (a.pair = P >= 2, 128-row slabs, no split): block t
// computes whole slabs [P t, P t + P) as one continuous weight stream (the
// packed tiles of consecutive slabs are contiguous).  Slab j accumulates in
// TMEM columns 32 (j % 2); the epilogue warps finish slab j while the ring
// streams slab j+1, and hand the columns back (tmem_empty) before slab j+2.
// Each slab is still one k-ordered accumulation, so the outputs are
// bit-identical to the one-slab records.  Modes: kGemvSiluMul (interleaved
// gate/up rows) and kGemvStore (e.g. the LM head).
template <int STAGES>
__device__ __forceinline__ void store_slab_epilogue(const BodyCtx& c, const GemvArgs& a, int slab, uint32_t col,
                                                    const float* rvec) {
    const int q = (ltid() >> 5) & 3, lane = ltid() & 31;
    uint32_t raw[32];
    tc::tmem_ld_32x32b_x32(c.tmem_base + ((uint32_t)(q * 32) << 16) + col, raw);
    tc::tmem_ld_wait();
    uint16_t* out = reinterpret_cast<uint16_t*>(a.out);
    const int n = slab * 128 + q * 32 + lane;
#pragma unroll 8
    for (int b = 0; b < 32; ++b) out[(size_t)b * a.N + n] = f_to_bf16(__uint_as_float(raw[b]) * rvec[b]);
}

template <int STAGES>
__device__ void gemv_multi(const BodyCtx& c, const GemvArgs& a, uint64_t* dbg) {
    using L = TcSmem<kGemvBN, STAGES, kTcBK, 128>;
    char* base = align1024(c.smem);
    const int nb = a.N / 128, KB = a.K / kTcBK;
    const int t = c.bx + c.gx * (c.by + c.gy * c.bz);
    const int s0 = a.pair * t, ns = min(a.pair, nb - s0), total = ns * KB;
    uint64_t* full = reinterpret_cast<uint64_t*>(base + L::kBarOff);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;  // [2] slab accumulator final
    uint64_t* tempty = tfull + 2;      // [2] its TMEM columns read (4 epilogue warps)
    float* red = reinterpret_cast<float*>(base + L::kBarOff + 256);  // [4][32]
    float* rv = red + 128;                                            // [32]
    const int warp = ltid() >> 5, lane = ltid() & 31;
    const char* a_packed = reinterpret_cast<const char*>(a.w_packed) + (size_t)s0 * KB * L::kABytes;
    if (ltid() == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int k = 0; k < 2; ++k) {
            tc::mbar_init(&tfull[k], 1);
            tc::mbar_init(&tempty[k], 4);
        }
        tc::fence_mbar_init();
    }
    body_sync();
    if (warp == 0 && lane == 0) {
        if (desc_fence_needed(c.st ? &a : nullptr)) tc::tma_fence_desc(&a.tmX);
        const uint64_t pol = tc::policy_evict_first();
        auto issue_a = [&](int i) {
            tc::bulk_g2s_hint(base + (i % STAGES) * L::kStageBytes, a_packed + (size_t)i * L::kABytes, L::kABytes,
                              &full[i % STAGES], pol);
        };
        auto issue_b = [&](int i) {
            tc::tma_load_2d(base + (i % STAGES) * L::kStageBytes + L::kABytes, &a.tmX, &full[i % STAGES],
                            (i % KB) * kTcBK, 0);
        };
        // weights stream while the previous launch finishes; X only after wait_prev
        const int pre = min(STAGES, total);
        for (int i = 0; i < pre; ++i) {
            tc::mbar_arrive_expect_tx(&full[i], L::kStageBytes);
            issue_a(i);
        }
        if (a.l2_pf_kb && total > pre && wait_prev_streamed(c)) {
            const uint32_t tot = min((uint32_t)(total - pre) * L::kABytes, (uint32_t)a.l2_pf_kb << 10);
            for (uint32_t off = 0; off < tot; off += L::kABytes)
                tc::bulk_prefetch_l2(a_packed + (size_t)pre * L::kABytes + off, min(L::kABytes, tot - off));
        }
        wait_prev(c);
        if (dbg) dbg[7] = globaltimer();
        for (int i = 0; i < pre; ++i) issue_b(i);
        for (int i = pre; i < total; ++i) {
            const int s = i % STAGES;
            tc::mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
            tc::mbar_arrive_expect_tx(&full[s], L::kStageBytes);
            issue_a(i);
            issue_b(i);
        }
    } else if (warp == 1 && lane == 0) {
        constexpr uint32_t idesc = tc::idesc_bf16_f32(128, kGemvBN);
        for (int i = 0; i < total; ++i) {
            const int j = i / KB, kk = i - j * KB, s = i % STAGES;
            if (kk == 0 && j >= 2) {
                tc::mbar_wait(&tempty[j & 1], ((j >> 1) - 1) & 1);  // slab j-2's columns read
                tc::tc_fence_after();
            }
            tc::mbar_wait(&full[s], (i / STAGES) & 1);
            tc::tc_fence_after();
            char* sa = base + s * L::kStageBytes;
            const uint64_t ad = tc::smem_desc_k_sw128(sa), bd = tc::smem_desc_k_sw128(sa + L::kABytes);
#pragma unroll
            for (int k = 0; k < kTcBK / 16; ++k)
                tc::mma_bf16(c.tmem_base + 32 * (j & 1), ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc,
                             !(kk == 0 && k == 0));
            tc::mma_commit(&empty[s]);
            if (kk == KB - 1) tc::mma_commit(&tfull[j & 1]);
        }
    } else if (warp >= 4) {
        const int q = warp & 3;
        if (ltid() == 128) wait_prev(c);  // acquire for the statistics of earlier launches
        epi_sync();
        float ss = 0.f;
        if (a.stats_in) {
            const float* st = reinterpret_cast<const float*>(a.stats_in);
#pragma unroll 8
            for (int p = q * a.P_in / 4; p < (q + 1) * a.P_in / 4; ++p) ss += __ldcg(st + p * 32 + lane);
        }
        red[q * 32 + lane] = ss;
        epi_sync();
        if (warp == 4)
            rv[lane] = a.stats_in ? rsqrtf((((red[lane] + red[32 + lane]) + red[64 + lane]) + red[96 + lane]) /
                                               (float)a.K + a.eps)
                                  : 1.f;
        epi_sync();
        for (int j = 0; j < ns; ++j) {
            tc::mbar_wait(&tfull[j & 1], (j >> 1) & 1);
            tc::tc_fence_after();
            if (dbg && ltid() == 128 && j < 2) dbg[1 + j] = globaltimer();
            if (j == ns - 1 && ltid() == 128) mark_streamed(c);  // every load of the block has landed
            if (a.mode == kGemvSiluMul) gemv_silu_pair_epilogue(c, a, s0 + j, 32u * (j & 1), rv);
            else store_slab_epilogue<STAGES>(c, a, s0 + j, 32u * (j & 1), rv);
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[j & 1]);
        }
    }
    if (dbg && ltid() == 128) dbg[5] = globaltimer();
    tc::tc_fence_before();
    body_sync();
    if (ltid() == 0)
        for (int k = 0; k < 2 * STAGES + 4; ++k) tc::mbar_inval(&full[k]);
    if (dbg && ltid() == 0) dbg[6] = globaltimer();
}

// BM = 128 or 64 weight rows per slab (M = 64: smaller blocks for the small
// projections; rows 16q..16q+15 sit in TMEM lanes 32q.. of epilogue warp q).
// Block -> work: classic split-K (a.sk = 0: t -> slab t % nb, split t / nb,
// S equal splits, split S-1 combines) or stream-K (a.sk = 1: the grid's G
// blocks take equal contiguous runs of the nb x KB (slab, k-block) units,
// so any grid size -- e.g. a multiple of the lanes at every quota -- is
// balanced; a run spans at most two slabs, host-checked).  Either way a
// slab's partials are summed in ascending k order by its last contributor:
// the order is a function of (N, K, grid) only, never of the schedule.
template <int BM, int STAGES>
__device__ __forceinline__ void gemv_body(const BodyCtx& c, const GemvArgs& a) {
    static_assert(TcSmem<kGemvBN, STAGES, kTcBK, BM>::kBarOff >= kGemvResOff + 32 * BM * 2,
                  "the staged residual inputs fit the consumed ring");
    constexpr int QR = BM / 4;            // slab rows per epilogue warp
    constexpr int FJ = BM * 8 / kBodyThreads;  // float4 per thread over a [BM][32] block
    char* base = align1024(c.smem);
    const int nb = a.N / BM;
    const int t = c.bx + c.gx * (c.by + c.gy * c.bz);
    const int KB = a.K / kTcBK;
    // pA: the block's first piece; pB (np = 2): the head of the next slab.
    // A run is at most KB k-blocks long (host-checked), so with two pieces pA
    // ends its slab (owner) and pB does not (non-owner).
    GemvPiece pA, pB{};
    int np = 1;
    if (a.sk) {
        const int G = c.gx * c.gy * c.gz;
        const int64_t U = (int64_t)nb * KB;
        const int64_t u0 = (int64_t)t * U / G, u1 = (int64_t)(t + 1) * U / G;
        const int n = (int)(u0 / KB), ka = (int)(u0 % KB);
        const int kb = (int)min((int64_t)KB, ka + (u1 - u0));
        const int first = gemv_block_of((int64_t)n * KB, U, G), last = gemv_block_of((int64_t)n * KB + KB - 1, U, G);
        pA = GemvPiece{n, ka, kb, t - first, last - first + 1, kb == KB};
        if (u0 + (kb - ka) < u1) {
            const int lastB = gemv_block_of((int64_t)(n + 1) * KB + KB - 1, U, G);
            pB = GemvPiece{n + 1, 0, (int)(u1 - (int64_t)(n + 1) * KB), 0, lastB - t + 1, false};
            np = 2;
        }
    } else {
        const int n = t % nb, s = t / nb;
        pA = GemvPiece{n, (int)((int64_t)s * KB / a.S), (int)((int64_t)(s + 1) * KB / a.S), s, a.S, s == a.S - 1};
    }
    uint64_t* dbg = a.dbg ? reinterpret_cast<uint64_t*>(a.dbg) + (size_t)t * 8 : nullptr;
    if (dbg && ltid() == 0) dbg[0] = globaltimer();
    BodyCtx cd = c;
    cd.dbg = dbg;
    // the owner's per-row RMSNorm scale, computed during the mainloop, lives
    // past the barriers (the ring is busy until the accumulators are final)
    float* rv_pre = reinterpret_cast<float*>(base + TcSmem<kGemvBN, STAGES, kTcBK, BM>::kBarOff + 256);
    gemv_mainloop<BM, STAGES>(base, a, pA, pB, np, c.tmem_base, cd, pA.owner ? rv_pre : nullptr);
    if (ltid() == 128) mark_streamed(c);  // tmem_full: every weight / X load of this block has landed
    wait_prev_all(c);  // the epilogue reads residual / norm statistics of earlier launches
    if (dbg && ltid() == 128) dbg[1] = globaltimer();
    const int warp = ltid() >> 5, lane = ltid() & 31;
    float* scratch = reinterpret_cast<float*>(base + kGemvScratch);  // [128][33] + row sums [4][32]
    const int q = warp & 3;
    const bool active = lane < QR;  // lanes holding a slab row (all of them at BM = 128)
    const int row = q * QR + lane;  // epilogue warps: row within the slab
    // ---- non-owner piece (at most one): fp32 partial out, fire-and-forget
    // arrival; before the owner piece's wait, so no block ever waits on a
    // block that is itself waiting
    const bool has_non = np == 2 || !pA.owner;
    if (has_non) {
        const GemvPiece& pn = np == 2 ? pB : pA;
        const uint32_t col = np == 2 ? 32u : 0u;
        if (warp >= 4) {
            uint32_t raw[32];  // the tcgen05.ld is warp-collective; rows past BM (lanes >= QR) unused
            tc::tmem_ld_32x32b_x32(c.tmem_base + ((uint32_t)(q * 32) << 16) + col, raw);
            tc::tmem_ld_wait();
            if (active) {
                float4* w = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.ws) +
                                                      ((size_t)pn.c * a.N + pn.n * BM + row) * 32);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    w[j] = make_float4(__uint_as_float(raw[4 * j]), __uint_as_float(raw[4 * j + 1]),
                                       __uint_as_float(raw[4 * j + 2]), __uint_as_float(raw[4 * j + 3]));
            }
        }
        body_sync();  // orders the CTA's partial stores before thread 0's release
        if (ltid() == 0)
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(reinterpret_cast<uint32_t*>(a.counters) + pn.n)
                         : "memory");
    }
    if (pA.owner) {
        const int n_blk = pA.n, S = pA.nc;
        const int n = n_blk * BM + row;
        // kGemvResid: the residual inputs (an earlier launch's output, ordered
        // by the wait_prev before the X loads) are fetched now into the
        // consumed ring, so their latency hides under the partial exchange;
        // each thread later reads back exactly the values it loaded
        uint16_t* resb = reinterpret_cast<uint16_t*>(base + kGemvResOff);
        if (a.mode == kGemvResid && warp >= 4 && active) {
            const uint16_t* __restrict__ res = reinterpret_cast<const uint16_t*>(a.resid);
#pragma unroll
            for (int h2 = 0; h2 < 32; h2 += 16) {
                uint16_t rv[16];
#pragma unroll
                for (int b = 0; b < 16; ++b) rv[b] = __ldcg(res + (size_t)(h2 + b) * a.N + n);
#pragma unroll
                for (int b = 0; b < 16; ++b) resb[(h2 + b) * BM + row] = rv[b];
            }
        }
        if (S > 1) {
            // the owner's own partial stays on chip: [128 rows][8 float4] in the
            // (consumed) ring, same element order as a workspace slab
            float4* own = reinterpret_cast<float4*>(base + kGemvOwnOff);
            uint32_t* ctr = reinterpret_cast<uint32_t*>(a.counters) + n_blk;
            if (warp >= 4) {
                uint32_t raw[32];
                tc::tmem_ld_32x32b_x32(c.tmem_base + ((uint32_t)(q * 32) << 16), raw);
                tc::tmem_ld_wait();
                if (active) {
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        own[row * 8 + j] = make_float4(__uint_as_float(raw[4 * j]), __uint_as_float(raw[4 * j + 1]),
                                                       __uint_as_float(raw[4 * j + 2]), __uint_as_float(raw[4 * j + 3]));
                }
            }
            if (ltid() == 0) {
                while (ld_acquire_u32(ctr) != (uint32_t)(S - 1)) {
                    if (tenant_failed(c)) break;  // a contributor that will never be claimed
                    __nanosleep(32);
                }
                *ctr = 0;  // at rest for the next launch (which only arrives after this one completes)
            }
            body_sync();
            if (dbg && ltid() == 0) dbg[2] = globaltimer() | (1ull << 63);
            // all 256 threads, coalesced: thread owns float4 f = ltid() + 256 j
            // of the slab's [BM rows][32] block; partials summed in the fixed
            // order c = 0..S-1 (ascending k), the owner's own last
            const float4* wsb = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(a.ws) +
                                                                (size_t)n_blk * BM * 32);
            const size_t sstride4 = (size_t)a.N * 8;
            float4 acc[FJ];
#pragma unroll
            for (int j = 0; j < FJ; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 3
            for (int sp = 0; sp < S; ++sp) {
                float4 x[FJ];
                if (sp < S - 1) {
#pragma unroll
                    for (int j = 0; j < FJ; ++j) x[j] = __ldcg(wsb + sp * sstride4 + ltid() + 256 * j);
                } else {
#pragma unroll
                    for (int j = 0; j < FJ; ++j) x[j] = own[ltid() + 256 * j];
                }
#pragma unroll
                for (int j = 0; j < FJ; ++j) {
                    acc[j].x += x[j].x;
                    acc[j].y += x[j].y;
                    acc[j].z += x[j].z;
                    acc[j].w += x[j].w;
                }
            }
            body_sync();  // every thread's TMEM-side reads of the stats scratch are done
#pragma unroll
            for (int j = 0; j < FJ; ++j) {
                const int f = ltid() + 256 * j;
                float* dst = scratch + (f >> 3) * 33 + (f & 7) * 4;
                dst[0] = acc[j].x;
                dst[1] = acc[j].y;
                dst[2] = acc[j].z;
                dst[3] = acc[j].w;
            }
            body_sync();
            if (dbg && ltid() == 0) dbg[3] = globaltimer();
        } else if (warp >= 4) {
            uint32_t raw[32];
            tc::tmem_ld_32x32b_x32(c.tmem_base + ((uint32_t)(q * 32) << 16), raw);
            tc::tmem_ld_wait();
            if (active) {
#pragma unroll
                for (int b = 0; b < 32; ++b) scratch[row * 33 + b] = __uint_as_float(raw[b]);
            }
        }
        // from here the slab's accumulators are scratch[row * 33 + b] (fp32,
        // summed in k order); each mode reads them element by element, so no
        // 32-register array stays live through the epilogue
        if (warp >= 4) {
            // RMSNorm of the input rows folded in as a per-row scale (rv_pre,
            // computed during the mainloop); x 1.0 (exact) without it
            float* red = scratch + 128 * 33 + 64;  // [4][32] (kGemvResid row sums)
            const float* rvec = rv_pre;
            epi_sync();  // every row's accumulators in scratch (pair modes read the neighbour row)
            const float* acc = scratch + row * 33;
            if (dbg && ltid() == 128) dbg[4] = globaltimer();
            if (a.mode == kGemvStore) {
                uint16_t* out = reinterpret_cast<uint16_t*>(a.out);
                if (active) {
#pragma unroll 8
                    for (int b = 0; b < 32; ++b) out[(size_t)b * a.N + n] = f_to_bf16(acc[b] * rvec[b]);
                }
            } else if (a.mode == kGemvResid) {
                uint16_t* __restrict__ out = reinterpret_cast<uint16_t*>(a.out);
                if (active) {
#pragma unroll
                    for (int h2 = 0; h2 < 32; h2 += 16) {
                        uint16_t rv[16];  // residual inputs staged before the exchange
#pragma unroll
                        for (int b = 0; b < 16; ++b) rv[b] = resb[(h2 + b) * BM + row];
#pragma unroll
                        for (int b = 0; b < 16; ++b) {
                            const uint16_t hb = f_to_bf16(bf16_to_f(rv[b]) + acc[h2 + b] * rvec[h2 + b]);
                            out[(size_t)(h2 + b) * a.N + n] = hb;
                            const float hr = bf16_to_f(hb);
                            scratch[row * 33 + h2 + b] = hr * hr;
                        }
                    }
                }
                epi_sync();
                {  // fixed-order sum over the slab's rows: 4 quarter sums, then in order
                    float ss = 0.f;
#pragma unroll 8
                    for (int r = q * QR; r < q * QR + QR; ++r) ss += scratch[r * 33 + lane];
                    red[q * 32 + lane] = ss;
                    epi_sync();
                    if (warp == 4)
                        reinterpret_cast<float*>(a.stats_out)[n_blk * 32 + lane] =
                            ((red[lane] + red[32 + lane]) + red[64 + lane]) + red[96 + lane];
                }
            } else if (a.mode == kGemvSiluMul && BM == 128) {
                // interleaved slab rows: 2i gate feature i, 2i+1 its up partner.
                // Both lanes of a pair work: the even lane takes batch rows
                // 0-15, the odd lane 16-31 (as gemv_silu_pair_epilogue; same
                // per-element arithmetic, so the same bits), 16 independent
                // iterations per lane instead of 32 on half the lanes
                uint16_t* out = reinterpret_cast<uint16_t*>(a.out);
                const int pr = row & ~1, b0 = (row & 1) * 16;
                const int f = n_blk * 64 + (row >> 1);
                const int F = a.N / 2;
#pragma unroll
                for (int b = b0; b < b0 + 16; ++b) {
                    const float g = scratch[pr * 33 + b] * rvec[b], u = scratch[(pr + 1) * 33 + b] * rvec[b];
                    out[(size_t)b * F + f] = f_to_bf16(silu_mul(g, u));
                }
            } else if (a.mode == kGemvQKV && active) {
                if (n < a.q_dim) {
                    uint16_t* out = reinterpret_cast<uint16_t*>(a.out);
#pragma unroll 8
                    for (int b = 0; b < 32; ++b) out[(size_t)b * a.q_dim + n] = f_to_bf16(acc[b] * rvec[b]);
                } else {
                    const bool is_k = n < a.q_dim + a.kv_dim;
                    const int m = n - a.q_dim - (is_k ? 0 : a.kv_dim);
                    const int h = m >> 7, d = m & 127;
                    const int nkv = a.kv_dim >> 7;
                    uint16_t* cache = reinterpret_cast<uint16_t*>(is_k ? a.kcache : a.vcache);
#pragma unroll 8
                    for (int b = 0; b < 32; ++b)
                        cache[(((size_t)b * nkv + h) * a.Lmax + a.pos) * 128 + d] = f_to_bf16(acc[b] * rvec[b]);
                }
            }
        }
    }
    if (dbg && ltid() == 128) dbg[5] = globaltimer();
    tc_teardown<kGemvBN, STAGES, kTcBK, BM>(base);
    if (ltid() == 0) tc::mbar_inval(reinterpret_cast<uint64_t*>(base + TcSmem<kGemvBN, STAGES, kTcBK, BM>::kBarOff) + 2 * STAGES + 1);
    if (dbg && ltid() == 0) dbg[6] = globaltimer();
}

__device__ void body_gemv_bf16(const BodyCtx& c) {
    const GemvArgs& a = *reinterpret_cast<const GemvArgs*>(c.args);
    if (a.pair >= 2) {
        // multi-slab records need 128-row packed slabs and a per-slab epilogue
        // (SiLU pairing or plain store); anything else is a malformed record:
        // the tenant fails alone instead of writing wrong outputs
        if ((a.mode != kGemvSiluMul && a.mode != kGemvStore) || a.bm == 64 || !a.w_packed || a.sk) {
            if (ltid() == 0) raise_fault(c, DS_FAULT_BAD_INPUT);
            return;
        }
        const int t = c.bx + c.gx * (c.by + c.gy * c.bz);
        gemv_multi<kGemvStages>(c, a, a.dbg ? reinterpret_cast<uint64_t*>(a.dbg) + (size_t)t * 8 : nullptr);
        return;
    }
    if (a.bm == 64) gemv_body<64, kGemvStages64>(c, a);
    else gemv_body<128, kGemvStages>(c, a);
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
// KV cache of L positions.  Logical block t -> (b, kv head h, split sp)
// (the decode tenant uses S = 1: one block per (b, h)); with S > 1 the
// splits' (m, l, O) merge in order 0..S-1 in the block that retires last.
// ---------------------------------------------------------------------------
struct AttnArgs {
    TmaDesc tmK;        // K cache rows [rows][128] bf16 as a 2-D view, box {64 dims, kAttnChunk rows}, SWIZZLE_128B
    TmaDesc tmV;        // V cache, same view
    uint64_t q;         // bf16 [32][32*128]
    uint64_t out;       // bf16 [32][32*128]
    uint64_t ws;        // fp32 [256][S][4][130]
    uint64_t counters;  // u32 [256]
    int32_t L, Lmax, S;
    float scale;        // 1/sqrt(128)
    uint64_t dbg;       // optional [grid][8] timestamps
    uint64_t kbase;     // K / V cache base (the tensor maps' global address), for L2 prefetch
    uint64_t vbase;
    int32_t l2_pf_kb;   // early start: KB of K and of V past the ring prefetched into L2 once the previous
                        // launch has streamed (0 = ring only)
    int32_t tc;         // 1: both products on tcgen05 with TMEM accumulators (body_attn_decode_tc)
};

static_assert(offsetof(AttnArgs, q) == 256 && offsetof(AttnArgs, L) == 288 && offsetof(AttnArgs, scale) == 300 &&
                  offsetof(AttnArgs, dbg) == 304 && offsetof(AttnArgs, kbase) == 312 &&
                  offsetof(AttnArgs, l2_pf_kb) == 328 && offsetof(AttnArgs, tc) == 332,
              "AttnArgs layout (mirrored in _abi.py)");

// KV positions per pipeline stage (one TMA box height).  A stage holds the
// chunk's K and V rows as four SWIZZLE_128B half-tiles [chunk][64 dims]
// (K dims 0-63, K 64-127, V 0-63, V 64-127): row r of a half-tile is one
// position, so 8 consecutive positions hit 8 distinct 16-B bank groups and
// every ldmatrix below is conflict-free.
#ifndef DS_ATTN_CHUNK
#define DS_ATTN_CHUNK 64
#endif
constexpr int kAttnChunk = DS_ATTN_CHUNK;
constexpr int kAttnWpc = kAttnChunk / 16;                  // warps per chunk (16 positions each)
constexpr int kAttnGroups = 8 / kAttnWpc;                  // chunk c is consumed by warp group c % groups
constexpr uint32_t kAttnHalf = kAttnChunk * 128;           // one [chunk][64] bf16 half-tile
constexpr uint32_t kAttnStage = 4 * kAttnHalf;             // K + V of one chunk
constexpr int kAttnStages = (96 * 1024) / kAttnStage;      // 3 x 32 KB (chunk 64) or 6 x 16 KB (chunk 32)
constexpr uint32_t kAttnBarOff = kAttnStages * kAttnStage;
constexpr uint32_t kAttnQOff = kAttnBarOff + 1024;           // Q^T B fragments [8 ks][2][8 heads][4 tq] u32 (4-7 zero)
constexpr uint32_t kAttnSmem = kAttnQOff + 2048;
static_assert(kAttnChunk == 32 || kAttnChunk == 64, "chunk of 32 or 64 positions");
static_assert(kAttnStages >= kAttnGroups + 1, "every group needs a stage in flight beyond the others'");

// byte address of (position r, dim d (multiple of 8)) of a K or V chunk
// (tile = the chunk's K or V half-tile pair)
__device__ __forceinline__ uint32_t kv_addr(uint32_t tile, int r, int d) {
    return tile + (d >> 6) * kAttnHalf + r * 128 + ((((d & 63) >> 3) ^ (r & 7)) << 4);
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ float ex2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t movm_t(uint32_t a) {
    uint32_t d;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
    return d;
}
// D = A(16x16 bf16, row) . B(16x8 bf16, col) + D, fp32 accumulate
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// ---------------------------------------------------------------------------
// GQA decode attention on tcgen05 (a.tc = 1).  Same blocks, chunking and
// K/V staging as body_attn_decode (3-stage ring of 64-position chunks, one
// smem row per position), but both products run on the 5th-gen tensor core
// with accumulators in TMEM:
//   S^T[64 pos][8]  = K[64 pos][128] . Q^T          M = 64, N = 8 (4 heads + 4 zero),
//                                                    A = the K tile (K-major), B = Q^T (K-major)
//   O_q^T[128][16] += V^T[128][16 pos] . P_q^T       M = 128, N = 16 (4 heads + 12 zero), K = 16,
//                                                    A = the V tile read MN-major (dims contiguous),
//                                                    B = P_q^T in smem (K-major, no swizzle)
// Softmax stream q (epilogue warp 4+q) owns positions 16q..16q+15 of every
// chunk: it reads its 16 S^T rows (TMEM lanes 32q..32q+15), keeps its own
// running max / sum per head and writes P_q^T; O_q accumulates in its own 16
// TMEM columns.  The running max is lazy: it moves (and O_q, l_q are
// rescaled) only when a chunk's max exceeds it by more than 2^8, so P stays
// in [0, 256] and most chunks need no rescale.  The four streams merge in
// stream order at the end.  Every decision depends on the data alone:
// deterministic, and bit-identical wherever the block runs.
// Roles: warp 0 lane 0 TMA producer, warp 1 lane 0 MMA issuer, warps 4-7
// softmax + O epilogue.
// ---------------------------------------------------------------------------
constexpr uint32_t kAtQOff = kAttnStages * kAttnStage;            // Q^T [2 atoms][8 rows][128 B]
constexpr uint32_t kAtPOff = kAtQOff + 2048;                      // P^T [2 bufs][4 streams][512 B]
constexpr uint32_t kAtBarOff = kAtPOff + 4096;                    // barriers + exchange words
constexpr uint32_t kAtSmem = kAtBarOff + 1024;
constexpr float kAtLazy = 8.f;                                    // log2 of the largest unnormalised P
static_assert(kAttnChunk == 64, "the tcgen05 attention stages 64-position chunks");

__device__ __forceinline__ uint64_t smem_desc_mn_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    // MN-major SWIZZLE_128B: 64 MN-elements per 128-B row, 8 K-rows per atom;
    // LBO = next 64 MN-elements, SBO = next 8 K-rows (cute make_umma_desc<MN>)
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
__device__ __forceinline__ uint64_t smem_desc_k_interleave(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    // K-major, no swizzle: core matrices of 8 rows x 16 B; LBO = next K
    // core matrix, SBO = next 8 rows
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__device__ void body_attn_decode_tc(const BodyCtx& c, const AttnArgs& a) {
    const int t = c.bx + c.gx * (c.by + c.gy * c.bz);
    const int bh = t % 256, sp = t / 256;
    const int b = bh >> 3, h = bh & 7;
    const int warp = ltid() >> 5, lane = ltid() & 31;
    const int p0 = (int)((int64_t)sp * a.L / a.S), p1 = (int)((int64_t)(sp + 1) * a.L / a.S);
    const int nch = (p1 - p0 + kAttnChunk - 1) / kAttnChunk;
    char* base = align1024(c.smem);
    const uint32_t sbase = tc::smem_u32(base);
    // K and V of a stage recycle separately: K after its chunk's QK, V after its PV
    uint64_t* fullK = reinterpret_cast<uint64_t*>(base + kAtBarOff);  // [3]
    uint64_t* fullV = fullK + kAttnStages;                            // [3]
    uint64_t* emptyK = fullV + kAttnStages;                           // [3]
    uint64_t* emptyV = emptyK + kAttnStages;                          // [3]
    uint64_t* s_full = emptyV + kAttnStages;                          // [2] S^T of a chunk in TMEM
    uint64_t* s_free = s_full + 2;                                   // [2] 4 softmax warps read it
    uint64_t* p_ready = s_free + 2;                                  // [2] P^T written, O rescaled
    uint64_t* o_done = p_ready + 2;                                  // [2] PV of a chunk complete
    float* xchg = reinterpret_cast<float*>(base + kAtBarOff + 256);  // [2][4 streams][8]: alpha (0 = none)
    float* fin = xchg + 64;                                          // [4 streams][8 heads][m, l]
    const uint32_t tS = c.tmem_base, tO = c.tmem_base + 32;          // S: 2 x 8 cols; O: 4 streams x 16 cols
    const int row0 = (b * 8 + h) * a.Lmax + p0;
#ifdef DS_ATTN_TRACE  // diagnostic build: per-chunk timeline (dbg stride 128 per block)
    uint64_t* dbg = a.dbg ? reinterpret_cast<uint64_t*>(a.dbg) + (size_t)t * 128 : nullptr;
#else
    uint64_t* dbg = a.dbg ? reinterpret_cast<uint64_t*>(a.dbg) + (size_t)t * 8 : nullptr;
#endif
    if (dbg && ltid() == 0) dbg[0] = globaltimer();
    auto issue_k = [&](int i) {
        const int s = i % kAttnStages;
        tc::mbar_arrive_expect_tx(&fullK[s], 2 * kAttnHalf);
        tc::tma_load_3d_hint(base + s * kAttnStage, &a.tmK, &fullK[s], 0, row0 + i * kAttnChunk, 0,
                             tc::policy_evict_first());
    };
    auto issue_v = [&](int i) {
        const int s = i % kAttnStages;
        tc::mbar_arrive_expect_tx(&fullV[s], 2 * kAttnHalf);
        tc::tma_load_3d_hint(base + s * kAttnStage + 2 * kAttnHalf, &a.tmV, &fullV[s], 0, row0 + i * kAttnChunk, 0,
                             tc::policy_evict_first());
    };
    auto issue = [&](int i) {
        issue_k(i);
        issue_v(i);
    };
    if (ltid() == 0) {
        for (int s = 0; s < kAttnStages; ++s) {
            tc::mbar_init(&fullK[s], 1);
            tc::mbar_init(&fullV[s], 1);
            tc::mbar_init(&emptyK[s], 1);
            tc::mbar_init(&emptyV[s], 1);
        }
        for (int k = 0; k < 2; ++k) {
            tc::mbar_init(&s_full[k], 1);
            tc::mbar_init(&s_free[k], 4);
            tc::mbar_init(&p_ready[k], 1);
            tc::mbar_init(&o_done[k], 1);
        }
        tc::fence_mbar_init();
        tc::tma_fence_desc(&a.tmK);
        tc::tma_fence_desc(&a.tmV);
        // early start: chunks entirely below L-1 are immutable this step
        const int pre = min(kAttnStages, nch);
        int pk = 0;
        while (pk < pre && p0 + (pk + 1) * kAttnChunk <= a.L - 1) issue(pk++);
        wait_prev(c);
        for (int i = pk; i < pre; ++i) issue(i);
    }
    body_sync();  // barriers initialised; thread 0's acquire (wait_prev) for the whole lane
    if (dbg && ltid() == 0) dbg[7] = globaltimer();
    {  // Q^T -> smem, K-major SWIZZLE_128B: row r = head (rows 4-7 zero), 16-B chunk j of
       // dims [64 a, 64 a + 64) at atom a, chunk j ^ r
        const int r = ltid() >> 5, j16 = (ltid() >> 1) & 15, half = ltid() & 1;  // 8 rows x 16 chunks of 16 B, 2 threads each
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (r < 4 && !half) {
            const uint4* q = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.q) + (size_t)b * 4096 +
                                                            (h * 4 + r) * 128);
            v = __ldcg(q + j16);
        }
        if (!half) {
            const int at = j16 >> 3, jj = j16 & 7;
            *reinterpret_cast<uint4*>(base + kAtQOff + at * 1024 + r * 128 + ((jj ^ r) << 4)) = v;
        }
        // P^T buffers: rows 4-15 (padding heads) stay zero
        for (int i = ltid(); i < 4096 / 16; i += kBodyThreads)
            reinterpret_cast<uint4*>(base + kAtPOff)[i] = make_uint4(0u, 0u, 0u, 0u);
    }
    tc::fence_proxy_async();  // generic smem writes (Q^T, P^T zeros) -> tensor-core reads
    body_sync();
    if (warp == 0 && lane == 0) {
        // ---- K producer: refill a K slot once its chunk's QK consumed it ----
        for (int i = kAttnStages; i < nch; ++i) {
            tc::mbar_wait(&emptyK[i % kAttnStages], ((i / kAttnStages) - 1) & 1);
            issue_k(i);
        }
    } else if (warp == 2 && lane == 0) {
        // ---- V producer: refill a V slot once its chunk's PV consumed it ----
        for (int i = kAttnStages; i < nch; ++i) {
            tc::mbar_wait(&emptyV[i % kAttnStages], ((i / kAttnStages) - 1) & 1);
            issue_v(i);
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer ----
        constexpr uint32_t idS = tc::idesc_bf16_f32(64, 8);
        constexpr uint32_t idO = tc::idesc_bf16_f32(128, 16) | (1u << 15);  // A (V^T) MN-major
        auto qk = [&](int ci) {
            const int s = ci % kAttnStages, sb = ci & 1;
            tc::mbar_wait(&fullK[s], (ci / kAttnStages) & 1);
            if (ci >= 2) tc::mbar_wait(&s_free[sb], ((ci >> 1) - 1) & 1);
            tc::tc_fence_after();
            const uint32_t kt = sbase + s * kAttnStage;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const uint64_t ad = tc::smem_desc_k_sw128(base + (kt - sbase) + (ks >> 2) * kAttnHalf) + (uint64_t)((ks & 3) * 2);
                const uint64_t bd = tc::smem_desc_k_sw128(base + kAtQOff + (ks >> 2) * 1024) + (uint64_t)((ks & 3) * 2);
                tc::mma_bf16(tS + 8 * sb, ad, bd, idS, ks != 0);
            }
            tc::mma_commit(&s_full[sb]);
            tc::mma_commit(&emptyK[s]);  // K of the stage consumed
#ifdef DS_ATTN_TRACE
            if (dbg && ci < 16) dbg[80 + ci] = globaltimer();
#endif
        };
        if (nch > 0) qk(0);
        for (int ci = 0; ci < nch; ++ci) {
            if (ci + 1 < nch) qk(ci + 1);  // S of the next chunk while softmax runs on this one
            const int s = ci % kAttnStages, sb = ci & 1;
            tc::mbar_wait(&p_ready[sb], (ci >> 1) & 1);
            tc::mbar_wait(&fullV[s], (ci / kAttnStages) & 1);
            tc::tc_fence_after();
            const uint32_t vt = sbase + s * kAttnStage + 2 * kAttnHalf;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                // A: V^T [128 dims][16 positions 16q..], MN-major: dims 0-63 | 64-127 are the two
                // half-tiles (LBO = one half-tile), 8 positions per 1-KB atom (SBO)
                const uint64_t ad = smem_desc_mn_sw128(vt + q * 2048, kAttnHalf, 1024);
                // B: P_q^T [16 rows][16 positions], no swizzle: [k half][2 row groups][8 rows][16 B]
                const uint64_t bd = smem_desc_k_interleave(sbase + kAtPOff + sb * 2048 + q * 512, 256, 128);
                tc::mma_bf16(tO + 16 * q, ad, bd, idO, ci != 0);
            }
            tc::mma_commit(&o_done[sb]);
            tc::mma_commit(&emptyV[s]);  // V of the stage consumed
#ifdef DS_ATTN_TRACE
            if (dbg && ci < 16) dbg[64 + ci] = globaltimer();
#endif
        }
    } else if (warp >= 4) {
        // ---- softmax stream q: positions 16q..16q+15 of every chunk ----
        const int q = warp - 4;
        const float scale2 = a.scale * 1.4426950408889634f;
        float m[4] = {kNegInf, kNegInf, kNegInf, kNegInf};  // lazy running max per head (log2 units)
        float l[4] = {0.f, 0.f, 0.f, 0.f};                  // this lane's share of the running sums
        for (int ci = 0; ci < nch; ++ci) {
            const int sb = ci & 1;
#ifdef DS_ATTN_TRACE
            const bool tr = dbg && ltid() == 128 && ci < 14;
            if (tr) dbg[8 + 4 * ci] = globaltimer();
#endif
            tc::mbar_wait(&s_full[sb], (ci >> 1) & 1);
#ifdef DS_ATTN_TRACE
            if (tr) dbg[9 + 4 * ci] = globaltimer();
#endif
            tc::tc_fence_after();
            uint32_t raw[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                         : "=r"(raw[0]), "=r"(raw[1]), "=r"(raw[2]), "=r"(raw[3]), "=r"(raw[4]), "=r"(raw[5]),
                           "=r"(raw[6]), "=r"(raw[7])
                         : "r"(tS + 8 * sb + ((uint32_t)(q * 32) << 16)));
            tc::tmem_ld_wait();
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&s_free[sb]);
            // lane < 16: position 16q + lane of the chunk (M = 64: rows 16q.. in lanes 32q..32q+15)
            const int pos = ci * kAttnChunk + 16 * q + lane;
            const bool ok = lane < 16 && p0 + pos < p1;
            float sv[4], cm[4];
#pragma unroll
            for (int hh = 0; hh < 4; ++hh) {
                sv[hh] = ok ? __uint_as_float(raw[hh]) * scale2 : kNegInf;
                cm[hh] = sv[hh];
            }
#pragma unroll
            for (int off = 1; off < 16; off <<= 1)
#pragma unroll
                for (int hh = 0; hh < 4; ++hh) cm[hh] = fmaxf(cm[hh], __shfl_xor_sync(0xffffffffu, cm[hh], off));
            // lazy max: move it only when the chunk exceeds it by > 2^kAtLazy
            bool move = false;
#pragma unroll
            for (int hh = 0; hh < 4; ++hh) move |= cm[hh] > m[hh] + kAtLazy;
            float al[4] = {1.f, 1.f, 1.f, 1.f};
            if (move) {
#pragma unroll
                for (int hh = 0; hh < 4; ++hh) {
                    const float nm = fmaxf(m[hh], cm[hh]);
                    al[hh] = m[hh] == kNegInf ? 0.f : ex2_ftz(m[hh] - nm);
                    m[hh] = nm;
                    l[hh] *= al[hh];
                }
            }
            // P_q^T (bf16): row = head, column = position; buffer sb was last read by PV(ci-2)
            if (ci >= 2) tc::mbar_wait(&o_done[sb], ((ci >> 1) - 1) & 1);
            char* pb = base + kAtPOff + sb * 2048 + q * 512;
            if (lane < 16) {
#pragma unroll
                for (int hh = 0; hh < 4; ++hh) {
                    const float pv = (sv[hh] == kNegInf || m[hh] == kNegInf) ? 0.f : ex2_ftz(sv[hh] - m[hh]);
                    l[hh] += pv;
                    const __nv_bfloat16 pbf = __float2bfloat16_rn(pv);
                    // [k half (lane / 8)][row group 0][row hh][16 B] + (lane % 8) * 2
                    *reinterpret_cast<__nv_bfloat16*>(pb + (lane >> 3) * 256 + hh * 16 + (lane & 7) * 2) = pbf;
                }
            }
            if (lane == 0) {
#pragma unroll
                for (int hh = 0; hh < 4; ++hh) xchg[(sb * 4 + q) * 8 + hh] = move ? al[hh] : 1.f;
                xchg[(sb * 4 + q) * 8 + 7] = move ? 1.f : 0.f;
            }
#ifdef DS_ATTN_TRACE
            if (tr) dbg[10 + 4 * ci] = globaltimer();
#endif
            tc::fence_proxy_async();  // P^T (generic writes) before the tensor core reads it
            epi_sync();               // every stream's P^T and rescale decision
            // rescale O of the streams whose max moved (all 4 warps: O_q spans every lane)
            bool any = false;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) any |= xchg[(sb * 4 + qq) * 8 + 7] != 0.f;
            if (any && ci >= 1) {
                tc::mbar_wait(&o_done[(ci - 1) & 1], ((ci - 1) >> 1) & 1);  // PV(ci-1) final
                tc::tc_fence_after();
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    if (xchg[(sb * 4 + qq) * 8 + 7] == 0.f) continue;
                    uint32_t o[16];
                    const uint32_t ta = tO + 16 * qq + ((uint32_t)(q * 32) << 16);
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
                                 : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]), "=r"(o[4]), "=r"(o[5]), "=r"(o[6]),
                                   "=r"(o[7]), "=r"(o[8]), "=r"(o[9]), "=r"(o[10]), "=r"(o[11]), "=r"(o[12]), "=r"(o[13]),
                                   "=r"(o[14]), "=r"(o[15])
                                 : "r"(ta));
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int hh = 0; hh < 4; ++hh) o[hh] = __float_as_uint(__uint_as_float(o[hh]) * xchg[(sb * 4 + qq) * 8 + hh]);
                    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
                                 ::"r"(ta), "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7]),
                                   "r"(o[8]), "r"(o[9]), "r"(o[10]), "r"(o[11]), "r"(o[12]), "r"(o[13]), "r"(o[14]), "r"(o[15])
                                 : "memory");
                }
                tc::tmem_st_wait();
            }
            tc::tc_fence_before();
            epi_sync();  // P^T of every stream written, every rescale stored
            if (warp == 4 && lane == 0) tc::mbar_arrive(&p_ready[sb]);
#ifdef DS_ATTN_TRACE
            if (tr) dbg[11 + 4 * ci] = globaltimer();
#endif
        }
        // ---- merge the four streams ----
#pragma unroll
        for (int hh = 0; hh < 4; ++hh) {
#pragma unroll
            for (int off = 1; off < 16; off <<= 1) l[hh] += __shfl_xor_sync(0xffffffffu, l[hh], off);
        }
        if (lane == 0) {
#pragma unroll
            for (int hh = 0; hh < 4; ++hh) {
                fin[(q * 8 + hh) * 2] = m[hh];
                fin[(q * 8 + hh) * 2 + 1] = l[hh];
            }
        }
        if (nch > 0) tc::mbar_wait(&o_done[(nch - 1) & 1], ((nch - 1) >> 1) & 1);
        tc::tc_fence_after();
        epi_sync();
        // thread: dim d = 32 (warp - 4) + lane, heads 0-3 (TMEM lanes are dims)
        uint32_t o[4][4];
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(o[qq][0]), "=r"(o[qq][1]), "=r"(o[qq][2]), "=r"(o[qq][3])
                         : "r"(tO + 16 * qq + ((uint32_t)(q * 32) << 16)));
        }
        tc::tmem_ld_wait();
        const int d = 32 * q + lane;
        float O[4], Ls[4], M[4];
#pragma unroll
        for (int hh = 0; hh < 4; ++hh) {
            M[hh] = kNegInf;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) M[hh] = fmaxf(M[hh], fin[(qq * 8 + hh) * 2]);
            O[hh] = 0.f;
            Ls[hh] = 0.f;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {  // stream order
                const float mq = fin[(qq * 8 + hh) * 2];
                const float f = mq == kNegInf ? 0.f : ex2_ftz(mq - M[hh]);
                Ls[hh] += fin[(qq * 8 + hh) * 2 + 1] * f;
                O[hh] += __uint_as_float(o[qq][hh]) * f;
            }
        }
        bool write_out = true;
        if (a.S > 1) {
            __shared__ int last_flag_t[2];
            float* ws = reinterpret_cast<float*>(a.ws) + ((size_t)bh * a.S + sp) * 4 * 130;
#pragma unroll
            for (int hh = 0; hh < 4; ++hh) {
                ws[hh * 130 + d] = O[hh];
                if (d == 0) {
                    ws[hh * 130 + 128] = M[hh];
                    ws[hh * 130 + 129] = Ls[hh];
                }
            }
            epi_sync();
            if (warp == 4 && lane == 0) {
                uint32_t tk;
                __threadfence();
                asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;"
                             : "=r"(tk) : "l"(reinterpret_cast<uint32_t*>(a.counters) + bh) : "memory");
                last_flag_t[body_lane()] = tk == (uint32_t)a.S - 1;
            }
            epi_sync();
            write_out = last_flag_t[body_lane()] != 0;
            if (write_out) {
                __threadfence();
                const float* wsb = reinterpret_cast<const float*>(a.ws) + (size_t)bh * a.S * 4 * 130;
#pragma unroll
                for (int hh = 0; hh < 4; ++hh) {
                    float MM = kNegInf;
                    for (int s2 = 0; s2 < a.S; ++s2) MM = fmaxf(MM, __ldcg(wsb + s2 * 4 * 130 + hh * 130 + 128));
                    float oo = 0.f, ll = 0.f;
                    for (int s2 = 0; s2 < a.S; ++s2) {  // fixed order
                        const float* src = wsb + s2 * 4 * 130 + hh * 130;
                        const float mw = __ldcg(src + 128);
                        const float f = mw == kNegInf ? 0.f : ex2_ftz(mw - MM);
                        ll += __ldcg(src + 129) * f;
                        oo += __ldcg(src + d) * f;
                    }
                    O[hh] = oo;
                    Ls[hh] = ll;
                }
                epi_sync();
                if (warp == 4 && lane == 0) reinterpret_cast<uint32_t*>(a.counters)[bh] = 0;
            }
        }
        if (write_out) {
            uint16_t* orow = reinterpret_cast<uint16_t*>(a.out) + (size_t)b * 4096 + (h * 4) * 128 + d;
#pragma unroll
            for (int hh = 0; hh < 4; ++hh) orow[hh * 128] = f_to_bf16(O[hh] / Ls[hh]);
        }
    }
    tc::tc_fence_before();
    body_sync();
    if (ltid() == 0) mark_streamed(c);
    if (dbg && ltid() == 0) dbg[6] = globaltimer();
    if (ltid() == 0)
        for (int k = 0; k < 4 * kAttnStages + 8; ++k) tc::mbar_inval(&fullK[k]);
}

// GQA decode attention on tensor cores, positions split across warps.
// Chunk c (kAttnChunk positions) lands by TMA in stage c % kAttnStages and is
// consumed by warp group c % kAttnGroups: each warp of the group owns 16 of
// its positions and runs, in registers,
//   S^T[16 pos][8] = K[16 pos][128] . Q^T      (M = positions, N = the kv
//                                               group's 4 query heads + 4 zero)
//   online softmax per head (max over the 16 positions by shuffles)
//   O^T[128][8]   += V^T[128][16 pos] . P^T    (P^T regrouped by movmatrix)
// so no scores cross warps and nothing waits on another warp except the
// stage refill.  Each warp keeps its own (m, l, O) over the positions it
// owned; at the end the 8 warps merge in warp order.  Deterministic: the
// position -> warp map, the chunk order and every reduction tree are fixed
// functions of (L, S, block).
__device__ void body_attn_decode(const BodyCtx& c) {
    const AttnArgs& a = *reinterpret_cast<const AttnArgs*>(c.args);
    if (a.tc) {
        body_attn_decode_tc(c, a);
        return;
    }
    const int t = c.bx + c.gx * (c.by + c.gy * c.bz);
    const int bh = t % 256, sp = t / 256;
    const int b = bh >> 3, h = bh & 7;
    const int warp = ltid() >> 5, lane = ltid() & 31;
    const int g = lane >> 2, tq = lane & 3;  // mma fragment coordinates
    const int grp = warp / kAttnWpc, sub = warp % kAttnWpc;
    const int p0 = (int)((int64_t)sp * a.L / a.S), p1 = (int)((int64_t)(sp + 1) * a.L / a.S);
    const int nch = (p1 - p0 + kAttnChunk - 1) / kAttnChunk;
    char* base = align1024(c.smem);
    const uint32_t sbase = tc::smem_u32(base);
    uint64_t* full = reinterpret_cast<uint64_t*>(base + kAttnBarOff);  // [kAttnStages]
    // chunk each stage holds or is loading (written by the issuer before
    // the TMA): groups run independently, so a consumer first waits for its
    // chunk to be issued into the stage, then on the stage's full barrier
    // with the exact phase parity (never a phase behind or two ahead)
    int* stage_chunk = reinterpret_cast<int*>(base + kAttnBarOff + 256);  // [kAttnStages] (shared-window accesses)
    // warps of the consuming group done with the stage; the last one refills it
    uint32_t* stage_done = reinterpret_cast<uint32_t*>(base + kAttnBarOff + 512);        // [kAttnStages]
    const int row0 = (b * 8 + h) * a.Lmax + p0;
#ifdef DS_ATTN_TRACE  // diagnostic build: per-chunk timeline (dbg stride 128 per block)
    uint64_t* dbg = a.dbg ? reinterpret_cast<uint64_t*>(a.dbg) + (size_t)t * 128 : nullptr;
#else
    uint64_t* dbg = a.dbg ? reinterpret_cast<uint64_t*>(a.dbg) + (size_t)t * 8 : nullptr;
#endif
    if (dbg && ltid() == 0) dbg[0] = globaltimer();
    auto issue = [&](int i) {
#ifdef DS_ATTN_TRACE
        if (dbg && i < 64) dbg[64 + i] = globaltimer();
#endif
        const int s = i % kAttnStages;
        char* st = base + s * kAttnStage;
        const uint64_t pol = tc::policy_evict_first();
        asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(tc::smem_u32(&stage_chunk[s])), "r"(i) : "memory");
        tc::mbar_arrive_expect_tx(&full[s], kAttnStage);
        tc::tma_load_3d_hint(st, &a.tmK, &full[s], 0, row0 + i * kAttnChunk, 0, pol);
        tc::tma_load_3d_hint(st + 2 * kAttnHalf, &a.tmV, &full[s], 0, row0 + i * kAttnChunk, 0, pol);
    };
    if (ltid() == 0) {
        for (int s = 0; s < kAttnStages; ++s) {
            tc::mbar_init(&full[s], 1);
            stage_chunk[s] = -1;
            stage_done[s] = 0u;
        }
        tc::fence_mbar_init();
        tc::tma_fence_desc(&a.tmK);
        tc::tma_fence_desc(&a.tmV);
        // Early start: the cache rows below L-1 are immutable for this step
        // (the preceding QKV launch appends position L-1 only), so their
        // stages stream while that launch finishes; the chunk holding L-1
        // and the query rows are read only after wait_prev (launch order +
        // acquire).
        const int pre = min(kAttnStages, nch);
        int pk = 0;
        while (pk < pre && p0 + (pk + 1) * kAttnChunk <= a.L - 1) issue(pk++);
        if (a.l2_pf_kb && nch > pk && wait_prev_streamed(c)) {
            // the rest of this block's K and V rows (contiguous, 256 B per
            // position) into L2 while the previous launch's epilogues run
            const char* kb = reinterpret_cast<const char*>(a.kbase) + ((size_t)row0 + pk * kAttnChunk) * 256;
            const char* vb = reinterpret_cast<const char*>(a.vbase) + ((size_t)row0 + pk * kAttnChunk) * 256;
            const uint32_t by = min((uint32_t)a.l2_pf_kb << 10, (uint32_t)(p1 - p0 - pk * kAttnChunk) * 256u);
            for (uint32_t off = 0; off < by; off += 16384) {
                tc::bulk_prefetch_l2(kb + off, min(16384u, by - off));
                tc::bulk_prefetch_l2(vb + off, min(16384u, by - off));
            }
        }
        wait_prev(c);
        for (int i = pk; i < pre; ++i) issue(i);
    }
    body_sync();  // carries thread 0's acquire (wait_prev) to the whole lane
    if (dbg && ltid() == 0) dbg[7] = globaltimer();
    // Q^T as the B operand of S^T = K . Q^T: B[k = dim][n = head g]; heads
    // g >= 4 are zero padding (N = 8).  The fragments live in smem, in
    // fragment order (registers are the executor's scarce resource: the
    // O^T accumulators take 32 of them), and are re-read per k-step.
    const uint32_t qs = sbase + kAttnQOff;
    {
        // thread i: head i >> 6, u32 i & 63 of that head's 128 dims -> (ks, j, tq);
        // rows of the padding heads 4-7 are zero, so a fragment is one plain load
        const int hq = ltid() >> 6, w = ltid() & 63;
        const uint32_t v = __ldcg(reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint16_t*>(a.q) +
                                                                    (size_t)b * 4096 + (h * 4 + hq) * 128) + w);
        const int ks = w >> 3, j = (w >> 2) & 1, q4 = w & 3;
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(qs + (((ks * 2 + j) * 8 + hq) * 4 + q4) * 4), "r"(v) : "memory");
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(qs + (((ks * 2 + j) * 8 + 4 + hq) * 4 + q4) * 4), "r"(0u) : "memory");
    }
    body_sync();
    const uint32_t qfb = qs + (g * 4 + tq) * 4;
    auto qfrag = [&](int ks, int j) -> uint32_t {
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(qfb + (ks * 2 + j) * 128));
        return v;
    };
    const float scale2 = a.scale * 1.4426950408889634f;  // softmax in base 2
    // this thread: heads 2tq, 2tq+1 (real for tq < 2); O^T rows 16 mt + g, + 8
    float m0 = kNegInf, m1 = kNegInf, l0 = 0.f, l1 = 0.f;
    float o[8][4];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
#pragma unroll
        for (int j = 0; j < 4; ++j) o[mt][j] = 0.f;
    const int pw = 16 * sub;  // this warp's positions within a chunk
    const int lr = lane & 7, lm = lane >> 3;
    // per-thread parts of the ldmatrix addresses (kv_addr with the k-step
    // folded in at compile time): row offset, and the swizzle term XORed
    // into the 16-B chunk index (row % 8 == lr since pw % 16 == 0)
    const uint32_t qk_row = (uint32_t)(pw + lr + 8 * (lm & 1)) * 128u, qk_y = (uint32_t)(((lm >> 1) ^ lr) & 7) << 4;
    const uint32_t pv_row = (uint32_t)(pw + lr + 8 * (lm >> 1)) * 128u, pv_y = (uint32_t)(((lm & 1) ^ lr) & 7) << 4;
    for (int ci = grp; ci < nch; ci += kAttnGroups) {
        const int s = ci % kAttnStages;
#ifdef DS_ATTN_TRACE
        const int tj = ci / kAttnGroups;
        const bool tr = dbg && ltid() == 0 && tj < 12;
        if (tr) dbg[8 + 4 * tj] = globaltimer();
#endif
        {  // shared-window spin (a generic volatile load would take the global path)
            const uint32_t sc = tc::smem_u32(&stage_chunk[s]);
            int cur;
            do {
                asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(cur) : "r"(sc) : "memory");
            } while (cur != ci);
        }
#ifdef DS_ATTN_TRACE
        if (tr) dbg[9 + 4 * tj] = globaltimer();
#endif
        tc::mbar_wait(&full[s], (ci / kAttnStages) & 1);
#ifdef DS_ATTN_TRACE
        if (tr) dbg[10 + 4 * tj] = globaltimer();
#endif
        const uint32_t kt = sbase + s * kAttnStage, vt = kt + 2 * kAttnHalf;
        // ---- S^T[16 pos][8] = K[pw..pw+15][:] . Q^T (two chains) ----
        float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int ks = 0; ks < 8; ks += 2) {
            uint32_t a0, a1, a2, a3, c0, c1, c2, c3;
            ldsm_x4(kt + (ks >> 2) * kAttnHalf + qk_row + ((((2 * ks) & 7) << 4) ^ qk_y), a0, a1, a2, a3);
            ldsm_x4(kt + ((ks + 1) >> 2) * kAttnHalf + qk_row + ((((2 * ks + 2) & 7) << 4) ^ qk_y), c0, c1, c2, c3);
            mma16816(sa, a0, a1, a2, a3, qfrag(ks, 0), qfrag(ks, 1));
            mma16816(sb2, c0, c1, c2, c3, qfrag(ks + 1, 0), qfrag(ks + 1, 1));
        }
        // (pos g | g+8, head 2tq | 2tq+1), in log2 units (exp(x) = 2^(x log2 e));
        // positions past the range masked
        const int valid = p1 - (p0 + ci * kAttnChunk) - pw;
        float sv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) sv[j] = (sa[j] + sb2[j]) * scale2;
        if (valid < 16) {
            if (g >= valid) sv[0] = sv[1] = kNegInf;
            if (g + 8 >= valid) sv[2] = sv[3] = kNegInf;
        }
        // ---- online softmax per head over the warp's 16 positions ----
        float c0m = fmaxf(sv[0], sv[2]), c1m = fmaxf(sv[1], sv[3]);
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
            c0m = fmaxf(c0m, __shfl_xor_sync(0xffffffffu, c0m, off));
            c1m = fmaxf(c1m, __shfl_xor_sync(0xffffffffu, c1m, off));
        }
        // a head with no valid position yet keeps max -inf: exponents
        // against 0 then give 2^-inf = 0 (never -inf - -inf)
        const float n0 = fmaxf(m0, c0m), n1 = fmaxf(m1, c1m);
        const float z0 = n0 == kNegInf ? 0.f : n0, z1 = n1 == kNegInf ? 0.f : n1;
        const float al0 = ex2_ftz(m0 - z0), al1 = ex2_ftz(m1 - z1);
        const float e0 = ex2_ftz(sv[0] - z0), e1 = ex2_ftz(sv[1] - z1);
        const float e2 = ex2_ftz(sv[2] - z0), e3 = ex2_ftz(sv[3] - z1);
        m0 = n0;
        m1 = n1;
        // per-thread partial row sums (positions g, g+8); reduced over g at the end
        l0 = l0 * al0 + (e0 + e2);
        l1 = l1 * al1 + (e1 + e3);
        if (!__all_sync(0xffffffffu, al0 == 1.f && al1 == 1.f)) {  // x 1.0 is exact: skipped when no max moved
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                o[mt][0] *= al0;
                o[mt][1] *= al1;
                o[mt][2] *= al0;
                o[mt][3] *= al1;
            }
        }
        // P^T as the B operand: B[k = pos 2tq..][n = head g] = transpose of
        // the (pos g, head 2tq..) fragment, per 8x8 half
        const uint32_t pb0 = movm_t(pack_bf16x2(e0, e1));
        const uint32_t pb1 = movm_t(pack_bf16x2(e2, e3));
        // ---- O^T[128][8] += V^T[:, pw..pw+15] . P^T ----
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
            uint32_t a0, a1, a2, a3;
            ldsm_x4_t(vt + (mt >> 2) * kAttnHalf + pv_row + ((((2 * mt) & 7) << 4) ^ pv_y), a0, a1, a2, a3);
            mma16816(o[mt], a0, a1, a2, a3, pb0, pb1);
        }
        __syncwarp();
#ifdef DS_ATTN_TRACE
        if (tr) dbg[11 + 4 * tj] = globaltimer();
#endif
        // the group's last warp to finish the stage refills it.  A relaxed
        // count suffices: a warp's ldmatrix reads of the stage returned
        // before its MMAs could issue, i.e. before its arrival
        if (lane == 0) {
            uint32_t n;
            asm volatile("atom.relaxed.cta.shared::cta.add.u32 %0, [%1], 1;"
                         : "=r"(n) : "r"(tc::smem_u32(&stage_done[s])) : "memory");
            if (n == kAttnWpc - 1) {
                stage_done[s] = 0u;
                if (ci + kAttnStages < nch) issue(ci + kAttnStages);
            }
        }
        __syncwarp();
    }
    // l over the 8 g-rows of the warp (fixed tree)
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, off);
        l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    body_sync();  // every stage consumed: the ring is scratch from here on
    if (ltid() == 0) mark_streamed(c);
    if (dbg && ltid() == 0) dbg[1] = globaltimer();
    // ---- merge the 8 warps in warp order ----
    // scratch: O_w [8 warps][4 heads][128 dims] fp32, m/l [8][4]
    float* Ow = reinterpret_cast<float*>(base);
    float* Mw = Ow + 8 * 4 * 128;
    float* Lw = Mw + 32;
    if (tq < 2) {
        float* ow = Ow + warp * 512;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
            ow[(2 * tq) * 128 + 16 * mt + g] = o[mt][0];
            ow[(2 * tq + 1) * 128 + 16 * mt + g] = o[mt][1];
            ow[(2 * tq) * 128 + 16 * mt + g + 8] = o[mt][2];
            ow[(2 * tq + 1) * 128 + 16 * mt + g + 8] = o[mt][3];
        }
        if (g == 0) {
            Mw[warp * 4 + 2 * tq] = m0;
            Mw[warp * 4 + 2 * tq + 1] = m1;
            Lw[warp * 4 + 2 * tq] = l0;
            Lw[warp * 4 + 2 * tq + 1] = l1;
        }
    }
    body_sync();
    // thread -> (head hq, dims 2j, 2j+1)
    const int hq = ltid() >> 6, j2 = 2 * (ltid() & 63);
    float M = kNegInf;
#pragma unroll
    for (int w = 0; w < 8; ++w) M = fmaxf(M, Mw[w * 4 + hq]);
    float Ls = 0.f, O0 = 0.f, O1 = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        const float mw = Mw[w * 4 + hq];
        const float f = mw == kNegInf ? 0.f : ex2_ftz(mw - M);
        Ls += Lw[w * 4 + hq] * f;
        O0 += Ow[w * 512 + hq * 128 + j2] * f;
        O1 += Ow[w * 512 + hq * 128 + j2 + 1] * f;
    }
    bool write_out = true;
    if (a.S > 1) {
        // this split's (O, M, L) to the workspace; the split that retires
        // last merges splits 0..S-1 in order
        __shared__ int last_flag_l[2];
        int& last_flag = last_flag_l[body_lane()];
        float* ws = reinterpret_cast<float*>(a.ws) + ((size_t)bh * a.S + sp) * 4 * 130 + hq * 130;
        ws[j2] = O0;
        ws[j2 + 1] = O1;
        if (j2 == 0) {
            ws[128] = M;
            ws[129] = Ls;
        }
        body_sync();
        if (ltid() == 0) {
            uint32_t tk;
            asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;"
                         : "=r"(tk) : "l"(reinterpret_cast<uint32_t*>(a.counters) + bh) : "memory");
            last_flag = tk == (uint32_t)a.S - 1;
        }
        body_sync();
        write_out = last_flag != 0;
        if (write_out) {
            __threadfence();
            const float* wsb = reinterpret_cast<const float*>(a.ws) + (size_t)bh * a.S * 4 * 130 + hq * 130;
            M = kNegInf;
            for (int s2 = 0; s2 < a.S; ++s2) M = fmaxf(M, __ldcg(wsb + s2 * 4 * 130 + 128));
            Ls = O0 = O1 = 0.f;
            for (int s2 = 0; s2 < a.S; ++s2) {  // fixed order
                const float* src = wsb + s2 * 4 * 130;
                const float mw = __ldcg(src + 128);
                const float f = (mw == kNegInf) ? 0.f : ex2_ftz(mw - M);
                Ls += __ldcg(src + 129) * f;
                O0 += __ldcg(src + j2) * f;
                O1 += __ldcg(src + j2 + 1) * f;
            }
            if (ltid() == 0) reinterpret_cast<uint32_t*>(a.counters)[bh] = 0;
        }
    }
    if (write_out) {
        const float inv = 1.f / Ls;
        uint16_t* orow = reinterpret_cast<uint16_t*>(a.out) + (size_t)b * 4096 + (h * 4 + hq) * 128;
        *reinterpret_cast<uint32_t*>(orow + j2) = pack_bf16x2(O0 * inv, O1 * inv);
    }
    body_sync();
    if (dbg && ltid() == 0) dbg[6] = globaltimer();
    if (ltid() == 0)
        for (int s = 0; s < kAttnStages; ++s) tc::mbar_inval(&full[s]);
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
    uint64_t stats;   // fp32 [1][32]: sum of squares of each gathered row (0 = skip); bitwise what
                      // DS_BODY_RMSNORM computes over the written row, one launch fewer per step
};

__device__ void body_embed(const BodyCtx& c) {
    const EmbedArgs& a = *reinterpret_cast<const EmbedArgs*>(c.args);
    const int b = c.bx;
    int tok = __ldcg(reinterpret_cast<const int*>(a.tokens) + b);
    if (tok < 0 || tok >= a.vocab) {
        // a token outside the vocabulary is a local exception of this tenant
        // (the gather would read outside the table); the row is clamped so
        // the block itself stays in bounds
        if (ltid() == 0) raise_fault(c, DS_FAULT_BAD_INPUT);
        tok = tok < 0 ? 0 : a.vocab - 1;
    }
    const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.table) + (size_t)tok * a.d);
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(a.h) + (size_t)b * a.d);
    float ss = 0.f;
    for (int i = ltid(); i < a.d / 8; i += kBodyThreads) {
        const uint4 v = __ldcs(src + i);
        dst[i] = v;
        // same per-thread order, tree and partial sum as body_rmsnorm
        uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float lo = __uint_as_float(w[j] << 16), hi = __uint_as_float(w[j] & 0xffff0000u);
            ss += lo * lo + hi * hi;
        }
    }
    if (a.stats) {
        const int warp = ltid() >> 5, lane = ltid() & 31;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        __shared__ float epart_l[2][8];
        float* part = epart_l[body_lane()];
        if (lane == 0) part[warp] = ss;
        body_sync();
        if (ltid() == 0) {
            float t = 0.f;
            for (int w = 0; w < 8; ++w) t += part[w];
            reinterpret_cast<float*>(a.stats)[b] = t;
        }
    }
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
#pragma unroll 4
    for (int v = va + 8 * (int)ltid(); v < vb; v += 8 * kBodyThreads) {  // 4 loads in flight per thread
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
