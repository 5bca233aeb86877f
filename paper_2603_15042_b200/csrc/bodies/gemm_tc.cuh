// tcgen05/TMEM/TMA tile engine and the two contraction tenants built on it.
//
//   D[BM x BN] (fp32, TMEM) = sum_k A[BM rows][k] . B[BN rows][k]   (both K-major, bf16)
//
// One logical block = one output tile (training GEMM) or one (row-slab,
// K-split) piece (decode GEMV).  Per block: warp 0 is the TMA producer
// (SWIZZLE_128B tiles into a STAGES-deep smem ring, mbarrier complete_tx),
// warp 1 issues tcgen05.mma (one elected thread, accumulator in TMEM,
// tcgen05.commit frees ring slots), warps 4-7 drain TMEM with tcgen05.ld in
// the epilogue.  The K loop order and the split-K combine order are fixed
// functions of the logical block index, so results are bit-identical wherever
// and whenever the block runs (solo or as a coroutine).
#pragma once
#include "common.cuh"
#include "tc_ptx.cuh"

namespace ds {

struct alignas(64) TmaDesc {
    uint64_t w[16];  // CUtensorMap (128 B), encoded on the host
};

constexpr int kTcBM = 128;
constexpr int kTcBK = 64;  // 64 bf16 = one 128-B swizzle row

template <int BN, int STAGES, int BK = kTcBK, int BM = kTcBM>
struct TcSmem {
    static constexpr uint32_t kABytes = BM * BK * 2;  // 16 KB at BM = 128, BK = 64
    static constexpr uint32_t kBBytes = BN * BK * 2;
    static constexpr uint32_t kStageBytes = kABytes + kBBytes;
    static constexpr uint32_t kBarOff = STAGES * kStageBytes;
    static constexpr uint32_t kBytes = kBarOff + 1024;  // barriers + epilogue scratch follow
};

__device__ __forceinline__ char* align1024(char* p) {
    return reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// Runs the mainloop for one logical block; on return (all 256 threads) the
// accumulator is in TMEM columns [tmem_base, tmem_base + BN) and the epilogue
// warps (4-7) have passed the tmem_full barrier.  Returns the smem base.
// a_packed != nullptr: the A operand is pre-packed in HBM as the SWIZZLE_128B
// smem image of consecutive [128 x 64] tiles (row slab a_row/128, k-block kb at
// ((a_row/128) * a_kblocks + kb) * 16 KB), fetched with one contiguous 16-KB
// bulk copy per stage instead of 128 strided row segments.
// BK = 64: SWIZZLE_128B tiles (one 128-B row per K block); BK = 32:
// SWIZZLE_64B tiles (half the bytes per stage, twice the stages in the same smem)
// BM = 128 (default) or 64: with M = 64 the accumulator's rows 16q..16q+15
// sit in TMEM lanes 32q..32q+15 (half sub-partitions).
// k-block at which an abandonable mainloop stopped (~0u: ran to the end), per lane
__device__ __forceinline__ volatile uint32_t* tc_stop_word() {
    __shared__ uint32_t stop[2];
    return &stop[body_lane()];
}

// An abandonable mainloop reads its SM's control word every kYieldCheckEvery
// k-blocks (~1.5 us of MMA at 128x256x64), one check ahead: p99 yields stay
// under 10 us for ~2 % of the tile's throughput (every 4: ~1 %, p99 ~11 us).
#ifndef DS_YIELD_CHECK_EVERY
#define DS_YIELD_CHECK_EVERY 2
#endif
constexpr int kYieldCheckEvery = DS_YIELD_CHECK_EVERY;

// when the producer decided to stop (diagnostics: abandoned attempts log it)
__device__ __forceinline__ volatile uint64_t* tc_stop_time_of(int l) {
    __shared__ uint64_t t[2];
    return &t[l];
}
__device__ __forceinline__ volatile uint64_t* tc_stop_time() { return tc_stop_time_of(body_lane()); }

// Descriptor fences: a launch record's tensor maps are immutable once
// registered, so a lane fences them (generic -> tensormap proxy) on its first
// block of a record and skips the fence on the record's later blocks.  Keyed
// by the record's args pointer; nullptr (solo grids) always fences.
__shared__ const void* g_desc_fenced[2];

__device__ __forceinline__ bool desc_fence_needed(const void* key) {
    if (!key) return true;
    if (g_desc_fenced[body_lane()] == key) return false;
    g_desc_fenced[body_lane()] = key;
    return true;
}

template <int BN, int STAGES, int BK = kTcBK, int BM = kTcBM>
__device__ __forceinline__ void tc_mainloop(char* base, const TmaDesc* tmA, const TmaDesc* tmB, int a_row, int b_row,
                                            int kb_begin, int kb_end, uint32_t tmem_base, bool a_evict_first,
                                            const char* a_packed = nullptr, int a_kblocks = 0,
                                            const BodyCtx* dep = nullptr, const BodyCtx* yc = nullptr,
                                            bool acc_init = false, uint32_t l2_pf_bytes = 0,
                                            const void* fence_key = nullptr, uint32_t l2_hint = 0) {
    using L = TcSmem<BN, STAGES, BK, BM>;
    uint64_t* full = reinterpret_cast<uint64_t*>(base + L::kBarOff);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    const int warp = ltid() >> 5, lane = ltid() & 31;
    if (ltid() == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(tmem_full, 1);
        tc::fence_mbar_init();
        *tc_stop_word() = ~0u;
    }
    body_sync();
    const int nkb = kb_end - kb_begin;
    if (warp == 0 && lane == 0) {
        if (desc_fence_needed(fence_key)) {
            if (!a_packed) tc::tma_fence_desc(tmA);
            tc::tma_fence_desc(tmB);
        }
        // l2_hint bits [1:0] A, [3:2] B: 0 default (A: a_evict_first ? first : last; B: none),
        // 1 evict_first, 2 evict_last, 3 evict_normal
        auto pick = [](uint32_t h, uint64_t dflt) {
            return h == 1 ? tc::policy_evict_first() : h == 2 ? tc::policy_evict_last() : h == 3 ? tc::policy_evict_normal() : dflt;
        };
        const uint64_t pol = pick(l2_hint & 3u, a_evict_first ? tc::policy_evict_first() : tc::policy_evict_last());
        const uint32_t hb = (l2_hint >> 2) & 3u;
        const uint64_t pol_b = hb ? pick(hb, 0ull) : 0ull;
        auto issue_a = [&](int i) {
            const int s = i % STAGES;
            char* sa = base + s * L::kStageBytes;
            if (a_packed)
                tc::bulk_g2s_hint(sa, a_packed + ((size_t)(a_row / BM) * a_kblocks + kb_begin + i) * L::kABytes,
                                  L::kABytes, &full[s], pol);
            else
                tc::tma_load_2d_hint(sa, tmA, &full[s], (kb_begin + i) * BK, a_row, pol);
        };
        auto issue_b = [&](int i) {
            const int s = i % STAGES;
            if (hb)
                tc::tma_load_2d_hint(base + s * L::kStageBytes + L::kABytes, tmB, &full[s], (kb_begin + i) * BK, b_row, pol_b);
            else
                tc::tma_load_2d(base + s * L::kStageBytes + L::kABytes, tmB, &full[s], (kb_begin + i) * BK, b_row);
        };
        // With a dependency, the A operand (weights, immutable) streams while
        // the previous launch finishes; B (its output) only after wait_prev.
        const int pre = dep ? min(STAGES, nkb) : 0;
        for (int i = 0; i < pre; ++i) {
            tc::mbar_arrive_expect_tx(&full[i % STAGES], L::kStageBytes);
            issue_a(i);
        }
        // ... and, once the previous launch has streamed all its operands
        // (its epilogues are running, HBM is idle), up to l2_pf_bytes more of
        // the (contiguous, pre-packed) weight range are prefetched into L2
        if (dep && a_packed && l2_pf_bytes && nkb > pre && wait_prev_streamed(*dep)) {
            const char* g0 = a_packed + ((size_t)(a_row / BM) * a_kblocks + kb_begin + pre) * L::kABytes;
            const uint32_t tot = min((uint32_t)(nkb - pre) * L::kABytes, l2_pf_bytes);
            for (uint32_t off = 0; off < tot; off += L::kABytes)
                tc::bulk_prefetch_l2(g0 + off, min(L::kABytes, tot - off));
        }
        if (dep) wait_prev(*dep);
        if (dep && dep->dbg) dep->dbg[7] = globaltimer();
        for (int i = 0; i < pre; ++i) issue_b(i);
        // abandonable: the SM's control word is loaded one k-block ahead of
        // its use, so the check costs no latency on the issue path
        unsigned long long cw = yc ? ctl_word_here(*yc) : 0ull;
        uint32_t ex = yc ? ld_volatile_u32(&yc->st->ctl.exit) : 0u;
        for (int i = pre; i < nkb; ++i) {
            const int s = i % STAGES;
            const uint32_t ph = (i / STAGES) & 1;
            if (i >= STAGES) tc::mbar_wait(&empty[s], ph ^ 1);
            if (yc && (i & (kYieldCheckEvery - 1)) == 0) {
                const bool stop = !serves_tenant(cw, yc->tenant) || ex != 0u;
                if (stop) {
                    // k-blocks < i are issued and will be multiplied; the MMA
                    // thread stops when it finds k-block i not loaded
                    tc_stop_time()[0] = globaltimer();
                    *tc_stop_word() = (uint32_t)i;
                    break;
                }
                // both words for the next check, issued now: their latency
                // hides under the next k-blocks' MMAs
                cw = ctl_word_here(*yc);
                ex = ld_volatile_u32(&yc->st->ctl.exit);
            }
            tc::mbar_arrive_expect_tx(&full[s], L::kStageBytes);
            issue_a(i);
            issue_b(i);
        }
    } else if (warp == 1 && lane == 0) {
        constexpr uint32_t idesc = tc::idesc_bf16_f32(BM, BN);
        for (int i = 0; i < nkb; ++i) {
            const int s = i % STAGES;
            const uint32_t ph = (i / STAGES) & 1;
            if (yc) {
                bool stopped = false;
                while (!tc::mbar_try_wait(&full[s], ph)) {
                    if ((uint32_t)i >= *tc_stop_word()) {  // never loaded: the tile stops before it
                        stopped = true;
                        break;
                    }
                }
                if (stopped) break;
            } else {
                tc::mbar_wait(&full[s], ph);
            }
            tc::tc_fence_after();
            char* sa = base + s * L::kStageBytes;
            char* sb = sa + L::kABytes;
            const uint64_t ad = BK == 64 ? tc::smem_desc_k_sw128(sa) : tc::smem_desc_k_sw64(sa);
            const uint64_t bd = BK == 64 ? tc::smem_desc_k_sw128(sb) : tc::smem_desc_k_sw64(sb);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
                // +32 B per K=16 step inside the 128-B swizzle row
                tc::mma_bf16(tmem_base, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc,
                             acc_init || (i | k) != 0);
            }
            tc::mma_commit(&empty[s]);
        }
        tc::mma_commit(tmem_full);
    }
    if (warp >= 4) {
        tc::mbar_wait(tmem_full, 0);
        tc::tc_fence_after();
    }
}

template <int BN, int STAGES, int BK = kTcBK, int BM = kTcBM>
__device__ __forceinline__ void tc_teardown(char* base) {
    using L = TcSmem<BN, STAGES, BK, BM>;
    tc::tc_fence_before();
    body_sync();
    if (ltid() == 0) {
        uint64_t* full = reinterpret_cast<uint64_t*>(base + L::kBarOff);
        for (int s = 0; s < 2 * STAGES + 1; ++s) tc::mbar_inval(&full[s]);
    }
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// ---------------------------------------------------------------------------
// Training GEMM tenant: C[M,N] (bf16) = A[M,K] . B[N,K]^T, fp32 accumulate.
// Tile 128 x BN (BN in {64, 128, 256}), optional split-K S: logical block
// t -> (tile = t / S, split = t % S); tiles follow a grouped raster so the
// concurrently running tiles share A/B panels in L2.  S > 1 writes each
// split's fp32 partial to a workspace and a DS_BODY_SPLITK_REDUCE launch
// folds them in fixed split order (deterministic wherever blocks run).
// ---------------------------------------------------------------------------
struct GemmArgs {
    TmaDesc tmA;  // A [M][K] bf16, box {64, 128}
    TmaDesc tmB;  // B [N][K] bf16, box {64, BN}
    uint64_t C;   // bf16 [M][N]
    int32_t M, N, K;
    int32_t group_m;
    int32_t bn;      // 0 or 256, 128, 64
    int32_t splits;  // split-K factor S (0/1 = none)
    uint64_t ws;     // fp32 [tiles][S][128][BN] when S > 1
    int32_t bk;      // 0 or 64: SWIZZLE_128B K blocks of 64; 32: SWIZZLE_64B K blocks of 32 (4-stage ring)
    int32_t tma_store;  // 1: epilogue stages the bf16 tile in smem and writes it with TMA stores (tmC)
    int32_t abandon;    // give the tile up within ~2 k-blocks when the SM is revoked: 1 re-runs it from
                        // k = 0 (fastest yield), 2 spills the accumulators and resumes at k (no lost work)
    int32_t l2_hint;    // L2 policy of the A / B operand loads (tc_mainloop's l2_hint; 0 = A evict_last, B none)
    int32_t tiles;      // 0/1: one output tile per logical block; T >= 2: T consecutive raster tiles per block
                        // (gemm_multi: BN 64 / 128, no split-K, not abandonable; same bits per tile)
    int32_t fuse_fold;  // S > 1: the last-arriving split of each tile folds the S partials in split order and
                        // stores bf16 C itself (no SPLITK_REDUCE launch); per-tile tickets follow the workspace
    TmaDesc tmC;        // C [M][N] bf16, box {64, 128}, SWIZZLE_128B
};
static_assert(offsetof(GemmArgs, tmC) == 320 && sizeof(GemmArgs) == 448, "GemmArgs layout (mirrored in _abi.py)");
// host-side validation of abandonable GEMMs reads these fields (runtime.cpp)
static_assert(offsetof(GemmArgs, l2_hint) == 308 && offsetof(GemmArgs, tiles) == 312, "GemmArgs tail (mirrored in _abi.py)");
static_assert(offsetof(GemmArgs, K) == kGemmArgsOffK && offsetof(GemmArgs, bk) == kGemmArgsOffBk &&
                  offsetof(GemmArgs, abandon) == kGemmArgsOffAbandon, "GemmArgs offsets (ds_device.cuh)");

constexpr int kGemmBN = 256;
constexpr int kGemmStages = kCtasPerSm == 2 ? 2 : 4;

__device__ __forceinline__ void gemm_tile_coords(const GemmArgs& a, int bn, int tile, int& m_blk, int& n_blk) {
    const int m_blocks = a.M / kTcBM, n_blocks = a.N / bn;
    const int gm = a.group_m > 0 ? a.group_m : 16;
    const int group_size = gm * n_blocks;
    const int g = tile / group_size;
    const int first_m = g * gm;
    const int rows = min(gm, m_blocks - first_m);
    const int r = tile % group_size;
    m_blk = first_m + r % rows;
    n_blk = r / rows;
}

template <int BN, int STAGES, int BK = kTcBK>
__device__ __forceinline__ void gemm_body_bn(const BodyCtx& c, const GemmArgs& a) {
    char* base = align1024(c.smem);
    const int t = c.bx + c.gx * (c.by + c.gy * c.bz);
    const int S = a.splits > 1 ? a.splits : 1;
    const int tile = t / S, sp = t % S;
    int m_blk, n_blk;
    gemm_tile_coords(a, BN, tile, m_blk, n_blk);
    const int kbs = a.K / BK;
    const int kb0 = (int)((int64_t)sp * kbs / S), kb1 = (int)((int64_t)(sp + 1) * kbs / S);
    const BodyCtx* yc = (a.abandon && c.st && c.abandon) ? &c : nullptr;
    const int warp = ltid() >> 5, lane = ltid() & 31;
    // resume a spilled tile: its fp32 accumulators back into TMEM, continue at k
    const uint32_t res = yc ? c.resume : 0u;
    int kb_start = kb0;
    if (res) {
        const int j = (int)(res & 0xffffu) - 1;
        kb_start = (int)(res >> 16);
        unsigned long long* ring = c.st->retry + (size_t)c.tenant * kRetryStride;
        if (warp >= 4) {
            const int q = warp & 3, row = q * 32 + lane;
            const float* src = c.st->save + ((size_t)c.st->tenants[c.tenant].save_base + j) * kSaveFloats + (size_t)row * BN;
#pragma unroll 1
            for (int ch = 0; ch < BN / 32; ++ch) {
                uint32_t v[32];
                const uint4* p4 = reinterpret_cast<const uint4*>(src + ch * 32);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint4 x = __ldcg(p4 + u);
                    v[4 * u] = x.x;
                    v[4 * u + 1] = x.y;
                    v[4 * u + 2] = x.z;
                    v[4 * u + 3] = x.w;
                }
                tc::tmem_st_32x32b_x32(c.tmem_base + ((uint32_t)(q * 32) << 16) + ch * 32, v);
            }
            tc::tmem_st_wait();
        }
        tc::tc_fence_before();
        body_sync();
        tc::tc_fence_after();
        if (ltid() == 0) atomicExch(ring + j, 0ull);  // spill consumed: the slot is free again
    }
    tc_mainloop<BN, STAGES, BK>(base, &a.tmA, &a.tmB, m_blk * kTcBM, n_blk * BN, kb_start, kb1, c.tmem_base, false,
                                nullptr, 0, nullptr, yc, res != 0u, 0, c.st ? c.args : nullptr,
                                (uint32_t)a.l2_hint);
    const bool gave_up = yc && *tc_stop_word() != ~0u;  // epilogue warps: ordered by tmem_full
    if (gave_up) {
        // abandoned: spill the accumulators (when there are any) so the tile
        // continues at k elsewhere; nothing is stored to C
        const uint32_t k_abs = (uint32_t)kb_start + *tc_stop_word();
        if (warp >= 4 && a.abandon == 2 && (res != 0u || k_abs > (uint32_t)kb0)) {
            __shared__ int spill_l[2];
            volatile int* spill = &spill_l[body_lane()];
            const int q = warp & 3;
            if (q == 0 && lane == 0) {
                unsigned long long* ring = c.st->retry + (size_t)c.tenant * kRetryStride;
                const int home = (int)((smid() * kLanes + body_lane()) % kRetrySlots);
                *spill = claim_retry_slot(ring, home, kRetryReserved, &c.st->ctl.exit);
            }
            epi_sync();
            const int j = *spill;
            if (j >= 0) {  // -1: the executor is exiting, nothing to resume
            const int row = q * 32 + lane;
            float* dst = c.st->save + ((size_t)c.st->tenants[c.tenant].save_base + j) * kSaveFloats + (size_t)row * BN;
#pragma unroll 1
            for (int ch = 0; ch < BN / 32; ++ch) {
                uint32_t v[32];
                tc::tmem_ld_32x32b_x32(c.tmem_base + ((uint32_t)(q * 32) << 16) + ch * 32, v);
                tc::tmem_ld_wait();
                uint4* p4 = reinterpret_cast<uint4*>(dst + ch * 32);
#pragma unroll
                for (int u = 0; u < 8; ++u) __stcg(p4 + u, make_uint4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]));
            }
            if (q == 0 && lane == 0) *c.ab_info = (uint32_t)(j + 1) | (k_abs << 16);
            }
        }
    } else if (warp >= 4 && S == 1 && a.tma_store) {
        // bf16 tile staged in the (consumed) ring as BN/64 SWIZZLE_128B
        // [128 rows][64 cols] sub-tiles (conflict-free 16-B chunk writes),
        // then one thread issues BN/64 bulk tensor stores
        const int q = warp & 3;
        const int r = q * 32 + lane;
#pragma unroll 1
        for (int ch = 0; ch < BN / 32; ++ch) {
            uint32_t v[32];
            tc::tmem_ld_32x32b_x32(c.tmem_base + ((uint32_t)(q * 32) << 16) + ch * 32, v);
            tc::tmem_ld_wait();
            char* sub = base + (ch >> 1) * 16384 + r * 128;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint4 o;
                o.x = pack_bf16x2(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1]));
                o.y = pack_bf16x2(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3]));
                o.z = pack_bf16x2(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5]));
                o.w = pack_bf16x2(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7]));
                const int chunk = (ch & 1) * 4 + j;
                *reinterpret_cast<uint4*>(sub + ((chunk ^ (r & 7)) << 4)) = o;
            }
        }
        tc::fence_proxy_async();  // generic smem writes -> async proxy
        epi_sync();
        if (q == 0 && lane == 0) {
            for (int sub = 0; sub < BN / 64; ++sub)
                tc::tma_store_2d(&a.tmC, base + sub * 16384, n_blk * BN + sub * 64, m_blk * kTcBM);
            tc::bulk_commit();
            tc::bulk_wait_all();  // global writes complete before the block retires
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
    } else if (warp >= 4) {
        const int q = warp & 3;
        if (S == 1) {
            const int row = m_blk * kTcBM + q * 32 + lane;
            __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(a.C);
            uint4* dst = reinterpret_cast<uint4*>(C + (size_t)row * a.N + n_blk * BN);
#pragma unroll 1
            for (int ch = 0; ch < BN / 32; ++ch) {
                uint32_t v[32];
                tc::tmem_ld_32x32b_x32(c.tmem_base + ((uint32_t)(q * 32) << 16) + ch * 32, v);
                tc::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint4 o;
                    o.x = pack_bf16x2(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1]));
                    o.y = pack_bf16x2(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3]));
                    o.z = pack_bf16x2(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5]));
                    o.w = pack_bf16x2(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7]));
                    dst[ch * 4 + j] = o;
                }
            }
        } else {
            // fp32 partial of this split: ws[tile][sp][row][BN]
            float* ws = reinterpret_cast<float*>(a.ws) + (((size_t)tile * S + sp) * kTcBM + q * 32 + lane) * BN;
            uint4* dst = reinterpret_cast<uint4*>(ws);
#pragma unroll 1
            for (int ch = 0; ch < BN / 32; ++ch) {
                uint32_t v[32];
                tc::tmem_ld_32x32b_x32(c.tmem_base + ((uint32_t)(q * 32) << 16) + ch * 32, v);
                tc::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 8; ++j) dst[ch * 8 + j] = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            }
            if (a.fuse_fold) {
                // ticket: the split that arrives last folds the tile (release:
                // this split's partial stores, fenced before the add; acquire:
                // the others', fenced after it), in split order 0..S-1 per
                // element -- the SPLITK_REDUCE body's order, so the same bits
                __shared__ int last_l[2];
                volatile int* last = &last_l[body_lane()];
                uint32_t* tickets = reinterpret_cast<uint32_t*>(reinterpret_cast<float*>(a.ws) +
                                                                (size_t)(a.M / kTcBM) * (a.N / BN) * S * kTcBM * BN);
                epi_sync();
                if (q == 0 && lane == 0) {
                    __threadfence();
                    const uint32_t old = atomicAdd(tickets + tile, 1u);
                    *last = old == (uint32_t)(S - 1);
                    if (old == (uint32_t)(S - 1)) {
                        __threadfence();
                        tickets[tile] = 0u;  // at rest for the record's next launch
                    }
                }
                epi_sync();
                if (*last) {
                    const int row = q * 32 + lane;
                    const float* src = reinterpret_cast<const float*>(a.ws) + ((size_t)tile * S * kTcBM + row) * BN;
                    __nv_bfloat16* Cr = reinterpret_cast<__nv_bfloat16*>(a.C) + (size_t)(m_blk * kTcBM + row) * a.N +
                                        n_blk * BN;
#pragma unroll 1
                    for (int col = 0; col < BN; col += 4) {
                        float4 acc = __ldcg(reinterpret_cast<const float4*>(src + col));
                        for (int s2 = 1; s2 < S; ++s2) {
                            const float4 p = __ldcg(reinterpret_cast<const float4*>(src + (size_t)s2 * kTcBM * BN + col));
                            acc.x += p.x;
                            acc.y += p.y;
                            acc.z += p.z;
                            acc.w += p.w;
                        }
                        uint2 o;
                        o.x = pack_bf16x2(acc.x, acc.y);
                        o.y = pack_bf16x2(acc.z, acc.w);
                        *reinterpret_cast<uint2*>(Cr + col) = o;
                    }
                }
            }
        }
    }
    tc_teardown<BN, STAGES, BK>(base);
    if (yc && ltid() == 0 && *tc_stop_word() != ~0u) *c.abandon = 1u;
}

// ---------------------------------------------------------------------------
// Multi-tile blocks (GemmArgs.tiles = T >= 2; BN 64 or 128, S = 1): logical
// block t computes raster tiles [T t, T t + T) as one continuous operand
// stream through the lane's ring.  Tile j accumulates in TMEM columns
// BN (j % 2); the epilogue warps drain tile j into a bf16 staging image and
// TMA-store it while the ring streams and the MMA issuer multiplies tile j+1,
// then hand the columns back (tempty) before tile j+2.  For the tall, short-K
// GEMMs of a convolution stream (K = 64 .. 576: one to nine k-blocks per tile)
// this removes the per-tile block overhead (claim, barrier set-up, pipeline
// fill, store drain) that otherwise costs more than the tile's bytes.  Every
// tile is the same k-ordered tcgen05 chain (same instruction descriptor, same
// smem descriptors, same k steps) as in gemm_body_bn, so C is bit-identical
// to the one-tile records wherever the blocks run.
// ---------------------------------------------------------------------------
template <int BN, int STAGES>
__device__ void gemm_multi(const BodyCtx& c, const GemmArgs& a) {
    using L = TcSmem<BN, STAGES>;
    static_assert(2 * BN <= 256, "two TMEM accumulators per lane");
    static_assert(L::kBytes + BN * 256 + 1024 <= kLaneSmem, "ring + staging fit the lane");
    char* base = align1024(c.smem);
    char* stage_c = base + L::kBytes;  // BN/64 SWIZZLE_128B [128][64] bf16 images (1024-aligned)
    const int tiles_total = (a.M / kTcBM) * (a.N / BN);
    const int t = c.bx + c.gx * (c.by + c.gy * c.bz);
    const int j0 = a.tiles * t, nt = min(a.tiles, tiles_total - j0);
    const int nkb = a.K / kTcBK, total = nt * nkb;
    uint64_t* full = reinterpret_cast<uint64_t*>(base + L::kBarOff);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;  // [2] tile accumulator final
    uint64_t* tempty = tfull + 2;      // [2] its TMEM columns read (4 epilogue warps)
    const int warp = ltid() >> 5, lane = ltid() & 31;
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
        if (desc_fence_needed(c.st ? c.args : nullptr)) {
            tc::tma_fence_desc(&a.tmA);
            tc::tma_fence_desc(&a.tmB);
        }
        const uint64_t pol = tc::policy_evict_last();
        int m_blk = 0, n_blk = 0;
        for (int i = 0; i < total; ++i) {
            const int j = i / nkb, kk = i - j * nkb, s = i % STAGES;
            if (kk == 0) gemm_tile_coords(a, BN, j0 + j, m_blk, n_blk);
            if (i >= STAGES) tc::mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
            char* sa = base + s * L::kStageBytes;
            tc::mbar_arrive_expect_tx(&full[s], L::kStageBytes);
            tc::tma_load_2d_hint(sa, &a.tmA, &full[s], kk * kTcBK, m_blk * kTcBM, pol);
            tc::tma_load_2d(sa + L::kABytes, &a.tmB, &full[s], kk * kTcBK, n_blk * BN);
        }
    } else if (warp == 1 && lane == 0) {
        constexpr uint32_t idesc = tc::idesc_bf16_f32(kTcBM, BN);
        for (int i = 0; i < total; ++i) {
            const int j = i / nkb, kk = i - j * nkb, s = i % STAGES;
            if (kk == 0 && j >= 2) {
                tc::mbar_wait(&tempty[j & 1], ((j >> 1) - 1) & 1);  // tile j-2's columns read
                tc::tc_fence_after();
            }
            tc::mbar_wait(&full[s], (i / STAGES) & 1);
            tc::tc_fence_after();
            char* sa = base + s * L::kStageBytes;
            const uint64_t ad = tc::smem_desc_k_sw128(sa), bd = tc::smem_desc_k_sw128(sa + L::kABytes);
#pragma unroll
            for (int k = 0; k < kTcBK / 16; ++k)
                tc::mma_bf16(c.tmem_base + BN * (j & 1), ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc,
                             (kk | k) != 0);
            tc::mma_commit(&empty[s]);
            if (kk == nkb - 1) tc::mma_commit(&tfull[j & 1]);
        }
    } else if (warp >= 4) {
        const int q = warp & 3, r = q * 32 + lane;
        for (int j = 0; j < nt; ++j) {
            int m_blk, n_blk;
            gemm_tile_coords(a, BN, j0 + j, m_blk, n_blk);
            if (j > 0) {
                if (q == 0 && lane == 0) tc::bulk_wait_read_all();  // tile j-1's stores have read the staging image
                epi_sync();
            }
            tc::mbar_wait(&tfull[j & 1], (j >> 1) & 1);
            tc::tc_fence_after();
#pragma unroll 1
            for (int ch = 0; ch < BN / 32; ++ch) {
                uint32_t v[32];
                tc::tmem_ld_32x32b_x32(c.tmem_base + ((uint32_t)(q * 32) << 16) + BN * (j & 1) + ch * 32, v);
                tc::tmem_ld_wait();
                char* sub = stage_c + (ch >> 1) * 16384 + r * 128;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    uint4 o;
                    o.x = pack_bf16x2(__uint_as_float(v[8 * u + 0]), __uint_as_float(v[8 * u + 1]));
                    o.y = pack_bf16x2(__uint_as_float(v[8 * u + 2]), __uint_as_float(v[8 * u + 3]));
                    o.z = pack_bf16x2(__uint_as_float(v[8 * u + 4]), __uint_as_float(v[8 * u + 5]));
                    o.w = pack_bf16x2(__uint_as_float(v[8 * u + 6]), __uint_as_float(v[8 * u + 7]));
                    const int chunk = (ch & 1) * 4 + u;
                    *reinterpret_cast<uint4*>(sub + ((chunk ^ (r & 7)) << 4)) = o;
                }
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[j & 1]);
            tc::fence_proxy_async();  // generic smem writes -> async proxy
            epi_sync();
            if (q == 0 && lane == 0) {
                for (int sub = 0; sub < BN / 64; ++sub)
                    tc::tma_store_2d(&a.tmC, stage_c + sub * 16384, n_blk * BN + sub * 64, m_blk * kTcBM);
                tc::bulk_commit();
            }
        }
        if (q == 0 && lane == 0) {
            tc::bulk_wait_all();  // global writes complete before the block retires
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
    }
    tc::tc_fence_before();
    body_sync();
    if (ltid() == 0)
        for (int k = 0; k < 2 * STAGES + 4; ++k) tc::mbar_inval(&full[k]);
}

__device__ void body_gemm_bf16(const BodyCtx& c) {
    const GemmArgs& a = *reinterpret_cast<const GemmArgs*>(c.args);
    if (a.tiles > 1) {  // host-validated: bn 64 / 128, splits 1, bk 64, TMA store, not abandonable
        if (a.bn == 64) gemm_multi<64, kCtasPerSm == 2 ? 3 : 6>(c, a);
        else gemm_multi<128, kCtasPerSm == 2 ? 2 : 4>(c, a);
        return;
    }
    if (a.bk == 32 && (a.bn == 0 || a.bn == 256)) {  // 4 x 24 KB stages per lane
        gemm_body_bn<kGemmBN, kCtasPerSm == 2 ? 4 : 8, 32>(c, a);
        return;
    }
    switch (a.bn) {
        case 64: gemm_body_bn<64, kCtasPerSm == 2 ? 4 : 8>(c, a); break;
        case 128: gemm_body_bn<128, kCtasPerSm == 2 ? 3 : 6>(c, a); break;
        default: gemm_body_bn<kGemmBN, kGemmStages>(c, a); break;
    }
}

// Split-K fold: block (tile, row group) sums the S fp32 partials of its rows
// in split order 0..S-1 and stores bf16.  rows = 16 (0: legacy) .. 128 rows
// per block, grid = tiles * 128 / rows: every element is the same s-ordered
// sum whatever the row grouping, so the grouping is a pure launch-shape choice
// (wider groups: fewer, larger blocks, less per-block overhead).
struct SplitkReduceArgs {
    uint64_t ws;  // fp32 [tiles][S][128][BN]
    uint64_t C;   // bf16 [M][N]
    int32_t M, N, K;
    int32_t group_m;
    int32_t bn;
    int32_t splits;
    int32_t rows;  // rows per block: 0 (= 16), 16, 32, 64 or 128
    int32_t pad;
};
static_assert(sizeof(SplitkReduceArgs) == 48, "SplitkReduceArgs layout (mirrored in _abi.py)");

__device__ void body_splitk_reduce(const BodyCtx& c) {
    const SplitkReduceArgs& r = *reinterpret_cast<const SplitkReduceArgs*>(c.args);
    const int t = c.bx + c.gx * (c.by + c.gy * c.bz);
    const int R = r.rows > 0 ? r.rows : 16, groups = kTcBM / R;
    const int tile = t / groups, rg = t - tile * groups;
    GemmArgs g;
    g.M = r.M;
    g.N = r.N;
    g.group_m = r.group_m;
    int m_blk, n_blk;
    gemm_tile_coords(g, r.bn, tile, m_blk, n_blk);
    const int S = r.splits, BN = r.bn;
    const float* ws = reinterpret_cast<const float*>(r.ws) + (size_t)tile * S * kTcBM * BN;
    __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(r.C);
    for (int idx = 4 * (int)ltid(); idx < R * BN; idx += 4 * kBodyThreads) {
        const int row = rg * R + idx / BN, col = idx % BN;
        const float* src = ws + (size_t)row * BN + col;
        const size_t stride = (size_t)kTcBM * BN;  // one split's partial
        float4 acc = __ldcg(reinterpret_cast<const float4*>(src));
        int s = 1;
        // 8 partials in flight per thread, then added in split order (the
        // same fp32 add sequence as one at a time)
        for (; s + 8 <= S; s += 8) {
            float4 p[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) p[u] = __ldcg(reinterpret_cast<const float4*>(src + (s + u) * stride));
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                acc.x += p[u].x;
                acc.y += p[u].y;
                acc.z += p[u].z;
                acc.w += p[u].w;
            }
        }
        for (; s < S; ++s) {
            const float4 p = __ldcg(reinterpret_cast<const float4*>(src + s * stride));
            acc.x += p.x;
            acc.y += p.y;
            acc.z += p.z;
            acc.w += p.w;
        }
        uint2 o;
        o.x = pack_bf16x2(acc.x, acc.y);
        o.y = pack_bf16x2(acc.z, acc.w);
        *reinterpret_cast<uint2*>(C + (size_t)(m_blk * kTcBM + row) * r.N + n_blk * BN + col) = o;
    }
}

}  // namespace ds
