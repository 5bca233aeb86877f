// Microbenchmark: legacy warp-level mma.sync m16n8k16 (bf16 -> fp32) latency
// and per-SM throughput on sm_100a, and ldmatrix latency.  Build:
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/mb_hmma.cu -o scripts/mb_hmma
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void k_mma(int iters, float* out, long long* cyc) {
    float d[CHAINS][4];
    for (int c = 0; c < CHAINS; ++c)
        for (int j = 0; j < 4; ++j) d[c][j] = 0.f;
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x3f80, b1 = a0 ^ 0x3f00;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
                "{%0, %1, %2, %3};"
                : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    long long t1 = clock64();
    float s = 0;
    for (int c = 0; c < CHAINS; ++c)
        for (int j = 0; j < 4; ++j) s += d[c][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int CHAINS>
void run(int warps, int iters) {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 148 * 8);
    k_mma<CHAINS><<<148, warps * 32>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double c = (double)h[0];
    double per_mma_warp = c / (iters * CHAINS);
    double sm_mma_per_cycle = (double)warps * iters * CHAINS / c;
    printf("{\"chains\": %d, \"warps_per_sm\": %d, \"cycles_per_mma_per_warp\": %.2f, \"sm_mma_per_cycle\": %.3f, "
           "\"sm_flop_per_cycle\": %.0f}\n",
           CHAINS, warps, per_mma_warp, sm_mma_per_cycle, sm_mma_per_cycle * 4096);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    const int it = 4096;
    run<1>(1, it);
    run<4>(1, it);
    run<8>(1, it);
    run<1>(4, it);
    run<4>(4, it);
    run<1>(8, it);
    run<4>(8, it);
    run<4>(16, it);
    run<8>(16, it);
    run<4>(32, it);
    return 0;
}
