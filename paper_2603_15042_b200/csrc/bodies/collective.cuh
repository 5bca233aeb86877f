// Gradient all-reduce of a data-parallel training tenant over NVLink peer
// memory, as an executor body (the only collective; it runs under
// the SM arbiter like any other logical block, so its SMs are charged to the
// training tenant's quota — a library collective's CTAs would bypass it).
//
// Every rank r of the DP group launches the same body over the same grid G
// after its gradient-producing launch.  Logical block b:
//   1. publishes "ready" for this epoch in its own flag line (release.sys) and
//      waits until every peer has published it (acquire.sys over NVLink);
//   2. sums chunk b of all W gradient buffers in rank order 0..W-1 in fp32
//      (peer loads over NVLink) and stores bf16 into its own output — every
//      rank computes the identical sum, bit for bit, in a fixed order;
//   3. counts itself done; the rank's last block waits until every peer has
//      counted G blocks, so no rank overwrites its gradient (next iteration)
//      while a peer still reads it.  Only the last block waits, so a rank's own
//      blocks can never be starved by its waiting blocks.
// The epoch is the launch sequence number (every rank of a DP tenant issues
// the same launch program); flag slots are epoch-tagged 64-bit words.
#pragma once
#include "common.cuh"

namespace ds {

constexpr int kMaxDpRanks = 8;
constexpr int kDpSlots = 64;
// flags of a rank: u64 ready[kDpSlots], done[kDpSlots], abort.  The host sets
// its own rank's abort word (ds_dp_abort) to release blocks still waiting for
// a peer that will never come (shutdown with a starved rank); results of an
// aborted launch are undefined, nothing hangs.
constexpr int kDpAbortWord = 2 * kDpSlots;

struct AllreduceArgs {
    uint64_t grad[kMaxDpRanks];   // bf16 [n] of rank p (peer-mapped pointers; own rank = local)
    uint64_t flags[kMaxDpRanks];  // u64 [2][kDpSlots] of rank p: ready, done
    uint64_t out;                 // bf16 [n], own
    int64_t n;                    // elements (multiple of 8)
    int32_t world, rank;
    int32_t chunk;                // elements per logical block (multiple of 8)
    int32_t pad;
};

__device__ __forceinline__ uint64_t ld_acquire_sys_u64_(const void* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ void body_allreduce_p2p(const BodyCtx& c) {
    const AllreduceArgs& a = *reinterpret_cast<const AllreduceArgs*>(c.args);
    const int b = c.bx + c.gx * (c.by + c.gy * c.bz);
    const int G = c.gx * c.gy * c.gz;
    const uint32_t epoch = c.seq + 1;  // nonzero
    const int slot = c.seq % kDpSlots;
    __shared__ int last_l[2];
    int& last = last_l[body_lane()];
    if (ltid() == 0) {
        unsigned long long* ready = reinterpret_cast<unsigned long long*>(a.flags[a.rank]) + slot;
        st_release_sys_u64(ready, epoch);
        for (int p = 0; p < a.world; ++p) {
            const void* pr = reinterpret_cast<const unsigned long long*>(a.flags[p]) + slot;
            while (ld_acquire_sys_u64_(pr) != epoch) {
                if (ld_volatile_u64(reinterpret_cast<const unsigned long long*>(a.flags[a.rank]) + kDpAbortWord)) break;
                if (tenant_failed(c)) break;
                __nanosleep(128);
            }
        }
    }
    body_sync();
    const int64_t i0 = (int64_t)b * a.chunk, i1 = min(a.n, i0 + a.chunk);
    for (int64_t i = i0 + 8 * (int64_t)ltid(); i < i1; i += 8 * kBodyThreads) {
        float acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.f;
        for (int p = 0; p < a.world; ++p) {  // fixed rank order
            const uint4 v = __ldcv(reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.grad[p]) + i));
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                acc[2 * j] += __uint_as_float(w[j] << 16);
                acc[2 * j + 1] += __uint_as_float(w[j] & 0xffff0000u);
            }
        }
        uint4 o;
        uint32_t* ow = &o.x;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t r;
            asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(acc[2 * j + 1]), "f"(acc[2 * j]));
            ow[j] = r;
        }
        *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(a.out) + i) = o;
    }
    __threadfence_system();
    body_sync();
    if (ltid() == 0) {
        // epoch-tagged done counter: (epoch << 32) | blocks done
        unsigned long long* done = reinterpret_cast<unsigned long long*>(a.flags[a.rank]) + kDpSlots + slot;
        unsigned long long w = *reinterpret_cast<volatile unsigned long long*>(done), nw;
        for (;;) {
            nw = ((w >> 32) == epoch) ? w + 1 : (((unsigned long long)epoch << 32) | 1ull);
            const unsigned long long old = atomicCAS(done, w, nw);
            if (old == w) break;
            w = old;
        }
        __threadfence_system();
        last = (int)(nw & 0xffffffffu) == G;
        if (last) {
            const unsigned long long want = ((unsigned long long)epoch << 32) | (unsigned long long)G;
            for (int p = 0; p < a.world; ++p) {
                const void* pd = reinterpret_cast<const unsigned long long*>(a.flags[p]) + kDpSlots + slot;
                while (ld_acquire_sys_u64_(pd) != want) {
                    if (ld_volatile_u64(reinterpret_cast<const unsigned long long*>(a.flags[a.rank]) + kDpAbortWord))
                        break;
                    if (tenant_failed(c)) break;
                    __nanosleep(256);
                }
            }
        }
    }
    body_sync();
}

}  // namespace ds
