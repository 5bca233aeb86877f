// Microbenchmark: per-lane / per-SM streaming rate of the GEMV ring
// (bulk copies into an smem ring; optional tcgen05 MMA consumer; optional
// L2 prefetch ahead of the ring).  Answers "what bounds a decode lane" apart
// from the executor.  Build: nvcc -O3 -std=c++17 -gencode
// arch=compute_100a,code=sm_100a -I paper_2603_15042_b200/csrc scripts/mb_stream.cu -o mb_stream
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include <cuda.h>
#include "bodies/tc_ptx.cuh"

using namespace ds;

struct alignas(64) TMap { CUtensorMap m; };
struct P {
    TMap xmap;          // X [32][K] bf16, box {64, 32}, SWIZZLE_128B (xtma = 1)
    int xtma;
    const char* src;
    const char* x;
    unsigned long long* t;   // [grid*lanes][2]
    size_t lane_bytes;
    int stages, lanes, mma, pf, wbytes, xbytes;
};

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
}

extern "C" __global__ void __launch_bounds__(128) k_stream(const __grid_constant__ P p) {
    extern __shared__ __align__(1024) char sm_raw[];
    char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    const int lane_id = threadIdx.x >> 6, w = (threadIdx.x >> 5) & 1, l = threadIdx.x & 31;
    if (lane_id >= p.lanes) return;
    const int stage_bytes = p.wbytes + p.xbytes;
    char* lb = base + lane_id * p.stages * stage_bytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + p.lanes * p.stages * stage_bytes) + lane_id * 64;
    uint64_t* full = bars;
    uint64_t* empty = bars + p.stages;
    __shared__ uint32_t tmem_slot[2];
    if (w == 1) {
        if (p.mma) tc::tmem_alloc(&tmem_slot[lane_id], 32);
        if (l == 0) {
            for (int s = 0; s < p.stages; ++s) {
                tc::mbar_init(&full[s], 1);
                tc::mbar_init(&empty[s], 1);
            }
            tc::fence_mbar_init();
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const int gl = blockIdx.x * p.lanes + lane_id;
    const char* src = p.src + (size_t)gl * p.lane_bytes;
    const int n = (int)(p.lane_bytes / p.wbytes);
    unsigned long long t0 = gt();
    if (w == 0 && l == 0) {
        const uint64_t pol = tc::policy_evict_first();
        for (int i = 0; i < n; ++i) {
            const int s = i % p.stages;
            if (i >= p.stages) tc::mbar_wait(&empty[s], ((i / p.stages) & 1) ^ 1);
            tc::mbar_arrive_expect_tx(&full[s], stage_bytes);
            char* d = lb + s * stage_bytes;
            tc::bulk_g2s_hint(d, src + (size_t)i * p.wbytes, p.wbytes, &full[s], pol);
            if (p.xbytes && p.xtma) tc::tma_load_2d(d + p.wbytes, &p.xmap, &full[s], (i & 63) * 64, 0);
            else if (p.xbytes) tc::bulk_g2s_hint(d + p.wbytes, p.x + (size_t)(i & 63) * p.xbytes, p.xbytes, &full[s],
                                                 tc::policy_evict_last());
            if (p.pf) {
                const size_t off = (size_t)i * p.wbytes + (size_t)p.pf;
                if (off < p.lane_bytes) tc::bulk_prefetch_l2(src + off, p.wbytes);
            }
        }
    } else if (w == 1 && l == 0) {
        const uint32_t idesc = tc::idesc_bf16_f32(128, 32);
        for (int i = 0; i < n; ++i) {
            const int s = i % p.stages;
            tc::mbar_wait(&full[s], (i / p.stages) & 1);
            if (p.mma) {
                tc::tc_fence_after();
                char* sa = lb + s * stage_bytes;
                const uint64_t ad = tc::smem_desc_k_sw128(sa), bd = tc::smem_desc_k_sw128(sa + p.wbytes);
                for (int k = 0; k < 4; ++k) tc::mma_bf16(tmem_slot[lane_id], ad + 2 * k, bd + 2 * k, idesc, (i | k) != 0);
                tc::mma_commit(&empty[s]);
            } else {
                tc::mbar_arrive(&empty[s]);
            }
        }
        if (p.mma) {
            // drain: last commit
            tc::mbar_wait(&empty[(n - 1) % p.stages], ((n - 1) / p.stages) & 1);
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (threadIdx.x % 64 == 0) {
        p.t[gl * 2] = t0;
        p.t[gl * 2 + 1] = gt();
    }
    if (w == 1 && p.mma) tc::tmem_dealloc(tmem_slot[lane_id], 32);
}

int main(int argc, char** argv) {
    // args: nsm lanes stages mma pf_kb xkb lane_mb
    int nsm = argc > 1 ? atoi(argv[1]) : 148;
    int lanes = argc > 2 ? atoi(argv[2]) : 2;
    int stages = argc > 3 ? atoi(argv[3]) : 5;
    int mma = argc > 4 ? atoi(argv[4]) : 0;
    int pf_kb = argc > 5 ? atoi(argv[5]) : 0;
    int xkb = argc > 6 ? atoi(argv[6]) : 4;
    int lane_mb = argc > 7 ? atoi(argv[7]) : 2;
    int wkb = argc > 8 ? atoi(argv[8]) : 16;
    int xtma = argc > 9 ? atoi(argv[9]) : 0;
    P p{};
    p.xtma = xtma;
    p.lane_bytes = (size_t)lane_mb << 20;
    p.stages = stages;
    p.lanes = lanes;
    p.mma = mma;
    p.pf = pf_kb << 10;
    p.wbytes = wkb << 10;
    p.xbytes = xkb << 10;
    size_t total = p.lane_bytes * nsm * lanes;
    char *src, *x;
    unsigned long long* t;
    cudaMalloc(&src, total + (64 << 20));
    cudaMemset(src, 0, total + (64 << 20));
    cudaMalloc(&x, 32 * 4096 * 2 + 64 * 8192);
    cudaMemset(x, 0, 32 * 4096 * 2 + 64 * 8192);
    cudaMalloc(&t, nsm * lanes * 16);
    p.src = src;
    p.x = x;
    if (xtma) {  // X [32][4096] bf16 view of the x buffer (64 k-blocks), box {64, 32}
        cuuint64_t dims[2] = {4096, 32};
        cuuint64_t strides[1] = {4096 * 2};
        cuuint32_t box[2] = {64, 32};
        cuuint32_t es[2] = {1, 1};
        CUresult r = cuTensorMapEncodeTiled(&p.xmap.m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, strides, box, es,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    }
    p.t = t;
    int smem = lanes * stages * (p.wbytes + p.xbytes) + lanes * 64 * 8 + 1024;
    smem = std::max(smem, 120 << 10);  // one CTA per SM
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    std::vector<unsigned long long> h(nsm * lanes * 2);
    double best = 0, lane_rate = 0;
    for (int rep = 0; rep < 4; ++rep) {
        k_stream<<<nsm, 128, smem>>>(p);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("err %s\n", cudaGetErrorString(e));
            return 1;
        }
        cudaMemcpy(h.data(), t, h.size() * 8, cudaMemcpyDeviceToHost);
        unsigned long long mn = ~0ull, mx = 0;
        double lr = 0;
        for (int i = 0; i < nsm * lanes; ++i) {
            mn = std::min(mn, h[2 * i]);
            mx = std::max(mx, h[2 * i + 1]);
            lr += (double)p.lane_bytes / (double)(h[2 * i + 1] - h[2 * i]);
        }
        double gbs = (double)total / (double)(mx - mn);
        if (gbs > best) {
            best = gbs;
            lane_rate = lr / (nsm * lanes);
        }
    }
    printf("{\"nsm\": %d, \"lanes\": %d, \"stages\": %d, \"wkb\": %d, \"xkb\": %d, \"mma\": %d, \"pf_kb\": %d, \"xtma\": %d, \"GBps\": %.1f, "
           "\"per_sm_GBps\": %.1f, \"lane_GBps\": %.1f}\n",
           nsm, lanes, stages, wkb, xkb, mma, pf_kb, xtma, best, best / nsm, lane_rate);
    return 0;
}
