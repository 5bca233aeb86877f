// SGEMM tenant (BASELINE config 1): fp32 C[M,N] = A[M,K] . B[K,N], row-major.
// Logical block (bx, by) owns the 64x64 tile at rows by*64, cols bx*64.  Each
// output is ONE fma chain in ascending k seeded with +0 (explicit __fmaf_rn,
// no contraction freedom), so the bits are a pure function of the inputs and
// identical to the CPU checker oracle/cnumlab.c:cn_sgemm_fma — whatever SM runs
// the tile and whenever it is preempted between tiles.
#pragma once
#include "common.cuh"

namespace ds {

struct SgemmArgs {
    uint64_t A, B, C;
    int32_t M, N, K;
    int32_t pad;
};

// Tile 64x64, K slab 32; thread (ty, tx) owns rows ty*4.., cols tx*4...  A is
// staged row-major (As[m][k], padded to 36) so a thread reads 4 k values of a
// row in one LDS.128 (its warp shares 2 rows: broadcast), B as Bs[k][n]; per 4
// k steps: 8 LDS.128 for 64 FFMA.  The next slab is prefetched into registers
// while the current one is consumed.  Every output is still one fma chain in
// ascending k.
constexpr int kSgA = 36;  // As row stride (floats): 16-B aligned rows, float4 stores conflict-free

__device__ void body_sgemm(const BodyCtx& c) {
    const SgemmArgs& a = *reinterpret_cast<const SgemmArgs*>(c.args);
    const float* __restrict__ A = reinterpret_cast<const float*>(a.A);
    const float* __restrict__ B = reinterpret_cast<const float*>(a.B);
    float* __restrict__ C = reinterpret_cast<float*>(a.C);
    const int row0 = c.by * 64, col0 = c.bx * 64;
    float* As = reinterpret_cast<float*>(c.smem);                 // [64][36]
    float* Bs = reinterpret_cast<float*>(c.smem) + 64 * kSgA;     // [32][64]
    const int tid = ltid();
    const int ty = tid / 16, tx = tid % 16;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
    // slab loads: A 64x32 and B 32x64 = 512 float4 each, 2 per thread
    float4 ra[2], rb[2];
    auto load = [&](int k0) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int idx = tid + r * 256;
            const int m = idx / 8, kq = idx % 8;
            ra[r] = __ldg(reinterpret_cast<const float4*>(A + (size_t)(row0 + m) * a.K + k0 + kq * 4));
            const int k = idx / 16, nq = idx % 16;
            rb[r] = __ldg(reinterpret_cast<const float4*>(B + (size_t)(k0 + k) * a.N + col0 + nq * 4));
        }
    };
    load(0);
    for (int k0 = 0; k0 < a.K; k0 += 32) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int idx = tid + r * 256;
            *reinterpret_cast<float4*>(As + (idx / 8) * kSgA + (idx % 8) * 4) = ra[r];
            *reinterpret_cast<float4*>(Bs + (idx / 16) * 64 + (idx % 16) * 4) = rb[r];
        }
        body_sync();
        if (k0 + 32 < a.K) load(k0 + 32);
#pragma unroll 2
        for (int k = 0; k < 32; k += 4) {
            float4 av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = *reinterpret_cast<const float4*>(As + (ty * 4 + i) * kSgA + k);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) bv[kk] = *reinterpret_cast<const float4*>(Bs + (k + kk) * 64 + tx * 4);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float x = kk == 0 ? av[i].x : kk == 1 ? av[i].y : kk == 2 ? av[i].z : av[i].w;
                    acc[i][0] = __fmaf_rn(x, bv[kk].x, acc[i][0]);
                    acc[i][1] = __fmaf_rn(x, bv[kk].y, acc[i][1]);
                    acc[i][2] = __fmaf_rn(x, bv[kk].z, acc[i][2]);
                    acc[i][3] = __fmaf_rn(x, bv[kk].w, acc[i][3]);
                }
            }
        }
        body_sync();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float4 v = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        *reinterpret_cast<float4*>(&C[(size_t)(row0 + ty * 4 + i) * a.N + col0 + tx * 4]) = v;
    }
}

// Test body: each logical block busy-waits `ns` and records where/when it ran.
struct SpinArgs {
    uint64_t out;  // per block: {smid, t0, t1} as 3 x u64
    uint64_t ns;
};

__device__ void body_spin(const BodyCtx& c) {
    const SpinArgs& a = *reinterpret_cast<const SpinArgs*>(c.args);
    if (ltid() == 0) {
        uint32_t blk = c.bx + c.gx * (c.by + c.gy * c.bz);
        uint64_t t0 = globaltimer();
        uint64_t t = t0;
        while (t - t0 < a.ns) t = globaltimer();
        uint64_t* o = reinterpret_cast<uint64_t*>(a.out) + 3 * (uint64_t)blk;
        o[0] = smid();
        o[1] = t0;
        o[2] = t;
    }
    body_sync();
}

}  // namespace ds
