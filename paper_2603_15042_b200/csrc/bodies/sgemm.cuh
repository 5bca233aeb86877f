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

__device__ void body_sgemm(const BodyCtx& c) {
    const SgemmArgs& a = *reinterpret_cast<const SgemmArgs*>(c.args);
    const float* __restrict__ A = reinterpret_cast<const float*>(a.A);
    const float* __restrict__ B = reinterpret_cast<const float*>(a.B);
    float* __restrict__ C = reinterpret_cast<float*>(a.C);
    const int row0 = c.by * 64, col0 = c.bx * 64;
    float (*As)[64 + 4] = reinterpret_cast<float (*)[64 + 4]>(c.smem);              // [32][68], As[k][m]
    float (*Bs)[64] = reinterpret_cast<float (*)[64]>(c.smem + 32 * 68 * sizeof(float));  // [32][64]
    const int tid = ltid();
    const int ty = tid / 16, tx = tid % 16;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
    for (int k0 = 0; k0 < a.K; k0 += 32) {
        // A tile 64x32 -> As[k][m]; 2048 floats, 8 per thread
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            int idx = tid + r * 256;
            int m = idx / 32, k = idx % 32;
            As[k][m] = A[(size_t)(row0 + m) * a.K + k0 + k];
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            int idx = tid + r * 256;
            int k = idx / 64, n = idx % 64;
            Bs[k][n] = B[(size_t)(k0 + k) * a.N + col0 + n];
        }
        body_sync();
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
            float av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[k][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[k][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(av[i], bv[j], acc[i][j]);
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
