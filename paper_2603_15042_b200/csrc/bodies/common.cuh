// Helpers shared by tenant bodies.  Bodies run on 256 threads and must use
// body_sync() (named barrier 1, 256 threads) instead of __syncthreads(): in
// the executor the CTA also holds a scheduler warp and a loader warp that
// never enter tenant code.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "../ds_device.cuh"

namespace ds {

// A CTA of the executor hosts kLanes independent worker lanes; lane L owns
// threads [256 L, 256 L + 256) for bodies.  Bodies see a lane-local thread id
// and lane-private named barriers, so the same body code runs in either lane
// and in the solo wrapper (lane 0).
__device__ __forceinline__ uint32_t body_lane() { return threadIdx.x >> 8; }
__device__ __forceinline__ uint32_t ltid() { return threadIdx.x & 255; }
__device__ __forceinline__ void body_sync() {
    asm volatile("bar.sync %0, 256;" ::"r"(body_lane() ? 8 : 1) : "memory");
}
__device__ __forceinline__ void epi_sync() {  // the 4 epilogue warps of a lane
    asm volatile("bar.sync %0, 128;" ::"r"(body_lane() ? 12 : 7) : "memory");
}

__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint32_t smid() {
    uint32_t s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    return s;
}

__device__ __forceinline__ uint32_t ld_volatile_u32(const void* p) {
    uint32_t v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t ld_volatile_u64(const void* p) {
    uint64_t v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const void* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const void* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t ld_acquire_sys_u64(const void* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(void* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_volatile_u32(void* p, uint32_t v) {
    asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys_u64(void* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Wait until every earlier launch of this tenant has completed (acquire).
// Single-thread form (the caller alone polls); see wait_prev_all.
__device__ __forceinline__ void wait_prev(const BodyCtx& c) {
    if (!c.prev_head) return;
    // gpu-scope acquire: later loads (incl. L1) observe every write the
    // completed launches released through their retire atomics
    while (ld_acquire_u32(c.prev_head) < c.seq) __nanosleep(32);
}

// All 256 body threads: one thread polls, the lane barrier carries its
// acquire to the others (so ~300 lanes x 256 threads never hammer one word).
__device__ __forceinline__ void wait_prev_all(const BodyCtx& c) {
    if (!c.prev_head) return;
    if (ltid() == 0) wait_prev(c);
    body_sync();
}

}  // namespace ds
