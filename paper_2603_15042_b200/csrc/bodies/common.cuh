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

// ---------------------------------------------------------------------------
// Local exceptions (reference apply_local_exception, engine.cpp:1049-1083)
// ---------------------------------------------------------------------------
// A failed tenant's claim word is parked at kDead: no SM claims another of its
// blocks, blocks already running finish (their in-launch waits give up, see
// tenant_failed), and its launches never complete.  Other tenants' claim
// words, rings and buffers are untouched, so they carry on bit-exactly.
__device__ __forceinline__ void kill_claim(DevTenant* T) {
    unsigned long long w = ld_volatile_u64(&T->claim);
    for (;;) {
        if ((uint32_t)w >= kDead) return;
        const unsigned long long o = atomicCAS(&T->claim, w, (w & 0xffffffff00000000ull) | kDead);
        if (o == w) return;
        w = o;
    }
}

// First raise wins; later raises (and injections) of the same tenant are no-ops.
__device__ inline void fault_tenant(DevState* st, int t, uint32_t code, uint32_t seq, uint32_t block) {
    DevTenant* T = &st->tenants[t];
    if (atomicCAS(&T->fault, 0u, code) != 0u) return;
    // fence.sc: pairs with the one in try_open/open_next (Dekker) so a launch
    // opened concurrently is re-killed by whichever side comes second
    __threadfence();
    kill_claim(T);
    HostFault* hf = &st->mailbox->faults[t];
    hf->seq = seq;
    hf->block = block;
    // launches before head completed intact; from head on, early-started
    // blocks may have stopped waiting for their predecessor (wait_prev), so
    // none of them counts as completed
    hf->head = ld_acquire_u32(&T->head);
    hf->t = globaltimer();
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(&hf->code), "r"(code) : "memory");
}

__device__ __forceinline__ bool tenant_failed(const BodyCtx& c) {
    return c.st && ld_volatile_u32(&c.st->tenants[c.tenant].fault) != 0u;
}

// Called by one thread of a block whose input is invalid (e.g. a token id
// outside the vocabulary): the tenant fails alone instead of faulting the
// shared executor.  The block itself must skip the invalid access.
__device__ __forceinline__ void raise_fault(const BodyCtx& c, uint32_t code) {
    if (!c.st) return;  // solo grid: nothing to contain
    fault_tenant(c.st, c.tenant, code, c.seq, c.bx + c.gx * (c.by + c.gy * c.bz));
}

// ---------------------------------------------------------------------------
// Abandonable blocks (sub-block yields): a body may give its block up when
// this SM no longer serves its tenant; the block re-runs from scratch later
// (same code, same inputs: bit-identical), so no partial state is kept.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool serves_tenant(unsigned long long cw, int tenant) {
    int32_t ow = (int32_t)(uint32_t)cw;
    if (ow >= 0) ow &= kCtlTenantMask;
    const int32_t ln = (int32_t)(uint32_t)(cw >> 32);
    return ow == tenant || ln == tenant;
}

__device__ __forceinline__ unsigned long long ctl_word_here(const BodyCtx& c) {
    return ld_volatile_u64(&c.st->ctl.word[smid()]);
}

// Claim a free retry-ring slot nearest `home` for `v` (linear probing over
// 8-slot windows read with 16-B loads; CAS only on slots seen free).  The ring
// holds at most one entry per worker lane of the tenant's single open launch
// (ds_start checks lanes <= kRetrySlots); a full ring waits for a pop, and
// gives up (-1) only when the executor is exiting.
__device__ inline int claim_retry_slot(unsigned long long* ring, int home, unsigned long long v,
                                       const uint32_t* exit_word) {
    for (;;) {
        for (int w = 0; w < kRetrySlots; w += 8) {
            const int base = ((home & ~1) + w) % kRetrySlots;  // even: 16-B aligned pairs
            unsigned long long x[8];
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const int j = (base + 2 * p) % kRetrySlots;
                asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];"
                             : "=l"(x[2 * p]), "=l"(x[2 * p + 1]) : "l"(ring + j) : "memory");
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int j = (base + e) % kRetrySlots;
                if (x[e] == 0ull && atomicCAS(ring + j, 0ull, v) == 0ull) return j;
            }
        }
        if (ld_volatile_u32(exit_word) != 0u) return -1;
        __nanosleep(256);  // ring full (more abandoned blocks than lanes): wait for a pop
    }
}

__device__ __forceinline__ bool revoked_here(const BodyCtx& c) {
    return ld_volatile_u32(&c.st->ctl.exit) != 0u || !serves_tenant(ctl_word_here(c), c.tenant);
}

// Wait until every earlier launch of this tenant has completed (acquire).
// Single-thread form (the caller alone polls); see wait_prev_all.  Gives up
// if the tenant failed (its earlier launch will never complete).
__device__ __forceinline__ void wait_prev(const BodyCtx& c) {
    if (!c.prev_head) return;
    // gpu-scope acquire: later loads (incl. L1) observe every write the
    // completed launches released through their retire atomics
    while (ld_acquire_u32(c.prev_head) < c.seq) {
        if (tenant_failed(c)) return;
        __nanosleep(32);
    }
}

// One thread of a block whose HBM streaming is done (its last operand load
// landed): counts it towards its launch's streamed word.  The completer of
// launch s-1 resets the word to (s << 32) before it publishes head = s, and a
// block of launch s streams only after it observed that head, so one
// fire-and-forget add per block suffices (no CAS round trips under contention).
__device__ __forceinline__ void mark_streamed(const BodyCtx& c) {
    if (!c.st) return;  // solo
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(&c.st->tenants[c.tenant].streamed) : "memory");
}

// Single thread, before wait_prev: waits until launch seq-1 has either
// completed (false) or streamed all its blocks (true: HBM is about to idle
// through its epilogues, so the caller's prefetch does not compete with it).
// False at once in solo mode, for the first launch, or when the previous
// launch's body does not mark.
__device__ __forceinline__ bool wait_prev_streamed(const BodyCtx& c) {
    if (!c.prev_head || !c.st || c.seq == 0) return false;
    const uint32_t p = c.seq - 1;
    const LaunchSlot* ps = &c.st->rings[(size_t)c.tenant * (c.st->ring_mask + 1) + (p & c.st->ring_mask)];
    const int pb = ld_volatile_u32(reinterpret_cast<const uint32_t*>(&ps->body));
    if (pb != DS_BODY_GEMV_BF16 && pb != DS_BODY_ATTN_DECODE) return false;
    const unsigned long long want = ((unsigned long long)p << 32) | ld_volatile_u32(&ps->grid);
    const unsigned long long* w = &c.st->tenants[c.tenant].streamed;
    for (;;) {
        if (ld_acquire_u32(c.prev_head) >= c.seq) return false;
        if (ld_volatile_u64(w) == want) return true;
        if (tenant_failed(c)) return false;
        __nanosleep(32);
    }
}

// All 256 body threads: one thread polls, the lane barrier carries its
// acquire to the others (so ~300 lanes x 256 threads never hammer one word).
__device__ __forceinline__ void wait_prev_all(const BodyCtx& c) {
    if (!c.prev_head) return;
    if (ltid() == 0) wait_prev(c);
    body_sync();
}

}  // namespace ds
