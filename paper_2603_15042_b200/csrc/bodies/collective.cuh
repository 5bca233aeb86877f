// Gradient all-reduce of a data-parallel training tenant over NVLink peer
// memory, as an executor body (the only collective; it runs under
// the SM arbiter like any other logical block, so its SMs are charged to the
// training tenant's quota — a library collective's CTAs would bypass it).
//
// Reduce-scatter + all-gather in one launch.  The n elements are G chunks;
// chunk c belongs to shard owner(c) (W contiguous chunk ranges).  Every rank
// r launches the same body over the same grid G; its logical block j takes
// chunk (lo_r + j) mod G, so a rank's own shard comes first in claim order.
//   owner chunk:  wait until every peer published "gradient ready" for this
//                 epoch, sum the chunk of all W gradients in rank order
//                 0..W-1 in fp32 (peer loads over NVLink), store bf16 into its
//                 own output, publish the chunk's epoch flag (release.sys);
//   other chunk:  wait for the owner's chunk flag (acquire.sys), copy the
//                 owner's bf16 result into its own output.
// Each element is summed once, by one rank, in rank order: the bits are those
// of a rank-ordered fp32 sum rounded once to bf16, on every rank.  NVLink reads
// per rank: (W-1) n/W gradient elements + (W-1) n/W results = 2 (W-1)/W n
// elements (1.75 n at W = 8; an all-read all-reduce moves (W-1) n).  Owner
// blocks never wait on another rank's blocks of the same launch, and they are
// claimed first on every rank, so the waits cannot cycle.
// Teardown: a block counts itself done; the rank's last block waits until
// every peer has counted G, so no rank overwrites its gradient or output
// (next epoch) while a peer still reads them.  The epoch is the launch
// sequence number (every rank of a DP tenant issues the same launch program);
// flag words are epoch-tagged, so nothing is ever reset.
#pragma once
#include "common.cuh"

namespace ds {

constexpr int kMaxDpRanks = 8;
constexpr int kDpSlots = 64;
// flags of a rank: u64 ready[kDpSlots], done[kDpSlots], abort, then the
// chunk words chunk[kDpMaxChunks] (epoch of the last published result).  The
// host sets its own rank's abort word (ds_dp_abort) to release blocks still
// waiting for a peer that will never come (shutdown with a starved rank);
// results of an aborted launch are undefined, nothing hangs.
constexpr int kDpAbortWord = 2 * kDpSlots;
constexpr int kDpChunkWord0 = 2 * kDpSlots + 8;
constexpr int kDpMaxChunks = 4096;

struct AllreduceArgs {
    uint64_t grad[kMaxDpRanks];   // bf16 [n] of rank p (peer-mapped pointers; own rank = local)
    uint64_t flags[kMaxDpRanks];  // u64 flag words of rank p (ready, done, abort, chunk epochs)
    uint64_t out;                 // bf16 [n], own
    uint64_t outs[kMaxDpRanks];   // bf16 [n] output of rank p (peer-mapped; outs[rank] == out)
    int64_t n;                    // elements (multiple of 8)
    int32_t world, rank;
    int32_t chunk;                // elements per logical block (multiple of 8)
    int32_t pad;
};
static_assert(offsetof(AllreduceArgs, out) == 128 && offsetof(AllreduceArgs, outs) == 136 &&
                  offsetof(AllreduceArgs, n) == 200 && offsetof(AllreduceArgs, rank) == 212 &&
                  offsetof(AllreduceArgs, chunk) == 216,
              "AllreduceArgs layout (mirrored in _abi.py)");

__device__ __forceinline__ uint64_t ld_acquire_sys_u64_(const void* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ bool dp_wait_epoch(const BodyCtx& c, const AllreduceArgs& a, const void* word,
                                              unsigned long long want, int sleep_ns) {
    while (ld_acquire_sys_u64_(word) != want) {
        if (ld_volatile_u64(reinterpret_cast<const unsigned long long*>(a.flags[a.rank]) + kDpAbortWord)) return false;
        if (tenant_failed(c)) return false;
        __nanosleep(sleep_ns);
    }
    return true;
}

__device__ void body_allreduce_p2p(const BodyCtx& c) {
    const AllreduceArgs& a = *reinterpret_cast<const AllreduceArgs*>(c.args);
    const int j = c.bx + c.gx * (c.by + c.gy * c.bz);
    const int G = c.gx * c.gy * c.gz;
    const uint32_t epoch = c.seq + 1;  // nonzero
    const int slot = c.seq % kDpSlots;
    // shard r = chunks [lo(r), lo(r+1)); this rank's own shard first
    auto lo = [&](int r) { return (int)((int64_t)r * G / a.world); };
    const int mine0 = lo(a.rank), mine1 = lo(a.rank + 1);
    const int ch = (mine0 + j) % G;
    const bool own = ch < mine1 && ch >= mine0;
    int owner = 0;
    while (owner + 1 < a.world && lo(owner + 1) <= ch) ++owner;
    __shared__ int last_l[2];
    int& last = last_l[body_lane()];
    if (ltid() == 0) {
        // publish this rank's gradient (every block, idempotent: the launch
        // runs after the gradient's launch completed, and a rank may own no
        // chunk at all when G < W)
        unsigned long long* ready = reinterpret_cast<unsigned long long*>(a.flags[a.rank]) + slot;
        if (ld_volatile_u64(ready) != epoch) st_release_sys_u64(ready, epoch);
        if (own) {
            // an owner reads every peer's gradient: wait until all published it
            for (int p = 0; p < a.world; ++p)
                if (!dp_wait_epoch(c, a, reinterpret_cast<const unsigned long long*>(a.flags[p]) + slot, epoch, 128)) break;
        } else {
            dp_wait_epoch(c, a, reinterpret_cast<const unsigned long long*>(a.flags[owner]) + kDpChunkWord0 + ch, epoch, 128);
        }
    }
    body_sync();
    const int64_t i0 = (int64_t)ch * a.chunk, i1 = min(a.n, i0 + a.chunk);
    uint16_t* out = reinterpret_cast<uint16_t*>(a.out);
    if (own) {
        for (int64_t i = i0 + 8 * (int64_t)ltid(); i < i1; i += 8 * kBodyThreads) {
            float acc[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[e] = 0.f;
            for (int p = 0; p < a.world; ++p) {  // fixed rank order
                const uint4 v = __ldcv(reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.grad[p]) + i));
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    acc[2 * e] += __uint_as_float(w[e] << 16);
                    acc[2 * e + 1] += __uint_as_float(w[e] & 0xffff0000u);
                }
            }
            uint4 o;
            uint32_t* ow = &o.x;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                uint32_t r;
                asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(acc[2 * e + 1]), "f"(acc[2 * e]));
                ow[e] = r;
            }
            *reinterpret_cast<uint4*>(out + i) = o;
        }
        __threadfence_system();
        body_sync();  // every thread's stores of the chunk before its flag
        if (ltid() == 0)
            st_release_sys_u64(reinterpret_cast<unsigned long long*>(a.flags[a.rank]) + kDpChunkWord0 + ch, epoch);
    } else {
        // gather the owner's result (NVLink peer loads, 16 B per thread)
        const uint16_t* src = reinterpret_cast<const uint16_t*>(a.outs[owner]);
        for (int64_t i = i0 + 8 * (int64_t)ltid(); i < i1; i += 8 * kBodyThreads)
            *reinterpret_cast<uint4*>(out + i) = __ldcv(reinterpret_cast<const uint4*>(src + i));
        __threadfence_system();
    }
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
            for (int p = 0; p < a.world; ++p)
                if (!dp_wait_epoch(c, a, reinterpret_cast<const unsigned long long*>(a.flags[p]) + kDpSlots + slot, want,
                                   256))
                    break;
        }
    }
    body_sync();
}

}  // namespace ds
