// Persistent GPU-coroutine executor + SM arbiter (sm_100a).
//
// One worker CTA per SM (cooperative launch, 1 CTA/SM forced by shared
// memory).  Each CTA reads %smid and, at every logical-block boundary, looks
// up the control word of its SM (owner tenant, then lender tenant), claims the
// next logical block of that tenant's current launch from the tenant's atomic
// claim word and runs the tenant's unmodified body on it.  Quota changes
// (host-written through the mailbox, or device-written by claim/time
// triggers) therefore take effect only at logical-block boundaries: an SM
// leaving a tenant finishes its current block first ("yield"), and the
// tenant's launch keeps its claim word, so it resumes — never restarts —
// wherever SMs are granted next (reference: signal_preempt /
// on_preempt_boundary / start_or_resume, src/engine/engine.cpp:756-806,925-984,470-529).
//
// Warp roles per CTA (320 threads):
//   warps 0-7  tenant body (256 threads, body_sync = named barrier 1)
//   warp 8     scheduler: claim -> stage -> (body runs) -> retire, logs
//   warp 9     CTA 0 only: loader — polls the host mailbox over PCIe, copies
//              launch slots into HBM rings, mirrors the control word.
#include <cuda_runtime.h>

#include <atomic>

#include "bodies/common.cuh"
#include "bodies/reduce.cuh"
#include "bodies/sgemm.cuh"
#include "bodies/gemm_tc.cuh"
#include "bodies/decode.cuh"
#include "bodies/collective.cuh"
#include "ds_device.cuh"

namespace ds {

constexpr uint32_t kTmemCols = 512;                  // whole TMEM, split between lanes
constexpr uint32_t kLaneTmemCols = kTmemCols / kLanes;

// ---------------------------------------------------------------------------
// Body dispatch (shared by the executor and the solo wrapper)
// ---------------------------------------------------------------------------
// Bodies that handle the early-start dependency themselves (stream immutable
// operands before wait_prev); every other body waits before it starts.
__device__ __forceinline__ bool early_start_body(int body) {
    return body == DS_BODY_GEMV_BF16 || body == DS_BODY_ATTN_DECODE;
}

// An abandonable GEMM block waiting for its tenant's previous launch gives
// itself up when its SM is revoked or when abandoned blocks wait in the
// tenant's retry ring (they may be the ones the previous launch needs: a
// waiting block must not hold the lane they could run on).  Abandonable
// tenants open a launch only once the previous one completed (try_claim), so
// this wait normally returns at once; it stays as a guard.
__device__ __forceinline__ bool wait_prev_or_abandon(const BodyCtx& c) {
    __shared__ uint32_t give_up_l[2];
    volatile uint32_t* give_up = &give_up_l[body_lane()];
    if (ltid() == 0) {
        uint32_t g = 0;
        while (ld_acquire_u32(c.prev_head) < c.seq) {
            if (tenant_failed(c)) break;
            if (ld_volatile_u32(&c.st->tenants[c.tenant].retry_count) != 0u || revoked_here(c)) {
                g = 1;
                break;
            }
            __nanosleep(64);
        }
        *give_up = g;
    }
    body_sync();
    const bool g = *give_up != 0u;
    body_sync();
    return !g;
}

__device__ __forceinline__ bool abandonable(int body, const BodyCtx& c) {
    return body == DS_BODY_GEMM_BF16 && c.abandon && reinterpret_cast<const GemmArgs*>(c.args)->abandon &&
           reinterpret_cast<const GemmArgs*>(c.args)->tiles <= 1;
}

__device__ __forceinline__ void run_body(int body, const BodyCtx& c) {
    if (!early_start_body(body)) {
        if (abandonable(body, c) && c.prev_head) {
            if (!wait_prev_or_abandon(c)) {
                if (ltid() == 0) {
                    *c.abandon = 1u;
                    if (c.resume) *c.ab_info = c.resume;  // hand the spill on untouched
                }
                return;
            }
        } else {
            wait_prev_all(c);
        }
    }
    switch (body) {
        case DS_BODY_REDUCE_CHUNKS: body_reduce(c); break;
        case DS_BODY_SGEMM: body_sgemm(c); break;
        case DS_BODY_SPIN: body_spin(c); break;
        case DS_BODY_GEMM_BF16: body_gemm_bf16(c); break;
        case DS_BODY_GEMV_BF16: body_gemv_bf16(c); break;
        case DS_BODY_ATTN_DECODE: body_attn_decode(c); break;
        case DS_BODY_RMSNORM: body_rmsnorm(c); break;
        case DS_BODY_EMBED: body_embed(c); break;
        case DS_BODY_ARGMAX: body_argmax(c); break;
        case DS_BODY_SPLITK_REDUCE: body_splitk_reduce(c); break;
        case DS_BODY_ALLREDUCE_P2P: body_allreduce_p2p(c); break;
        case DS_BODY_CHECKSUM: body_checksum(c); break;
        default: break;
    }
}

struct Stage {
    int32_t tenant;   // -1 exit
    int32_t body;
    uint32_t seq;
    uint32_t block;
    uint32_t gx, gy, gz;
    uint32_t pad;
    uint64_t args;
};

// ---------------------------------------------------------------------------
// Claim-word protocol
// ---------------------------------------------------------------------------
// Open launch `seq` if it is enqueued and its word is still closed.  Called by
// the completer of seq-1 and by the loader after publishing a new tail (the
// two sides are ordered by fence.sc, Dekker-style, so one of them opens it).
// A failed tenant never reopens: the fault word is checked before, and after
// a fence.sc past, the CAS (fault_tenant sets the word, fences, then kills).
__device__ __forceinline__ LaunchSlot* slot_of(DevState* st, int t, uint32_t s) {
    return &st->rings[(size_t)t * (st->ring_mask + 1) + (s & st->ring_mask)];
}

// First logical block of launch s: 0, or the resume point of a launch whose
// lower blocks ran on another device before a migration (ds_launch_from; the
// slot's flags word, written before the tail that publishes the slot).
__device__ __forceinline__ uint32_t first_block(DevState* st, int t, uint32_t s) {
    return ld_volatile_u32(&slot_of(st, t, s)->flags);
}

__device__ void try_open(DevState* st, int t) {
    DevTenant* T = &st->tenants[t];
    for (;;) {
        if (ld_volatile_u32(&T->fault)) return;
        unsigned long long w = ld_volatile_u64(&T->claim);
        uint32_t s = (uint32_t)(w >> 32), b = (uint32_t)w;
        if (b < kSat) return;
        uint32_t tail = ld_acquire_u32(&T->tail);
        if (s >= tail) return;
        if (atomicCAS(&T->claim, w, ((unsigned long long)s << 32) | first_block(st, t, s)) == w) {
            __threadfence();
            if (ld_volatile_u32(&T->fault)) kill_claim(T);
            return;
        }
    }
}

__device__ void log_ctl(DevState* st, uint32_t gen, uint32_t source) {
    if (st->clog_cap == 0) return;
    unsigned long long i = atomicAdd(&st->clog_count, 1ull);
    if (i < st->clog_cap) {
        ds_ctl_record r;
        r.ctl_gen = gen;
        r.source = source;
        r.t = globaltimer();
        st->clog[i] = r;
    }
}

// Lane-parallel install of a control word (owner/lender by smid).  All of a
// lane's source loads are issued before any store (one PCIe round trip when
// the source is the host mailbox); the control record is stamped when the
// install starts.
__device__ void install_ctl(DevState* st, const int32_t* owner, const int32_t* lender, bool volatile_src,
                            uint32_t source, int lane) {
    constexpr int kPer = DS_MAX_SMS / 32;
    const uint64_t t0 = globaltimer();
    if (lane == 0) asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(&st->ctl.t_install), "l"(t0) : "memory");
    int32_t o[kPer], l[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const int i = lane + 32 * j;
        if (volatile_src) {  // relaxed loads all in flight; one acquire fence below
            o[j] = (int32_t)ld_volatile_u32(owner + i);
            l[j] = (int32_t)ld_volatile_u32(lender + i);
        } else {
            o[j] = owner[i];
            l[j] = lender[i];
        }
    }
    // (host-image loads are ordered after the generation that announced
    // them by the loader's poll fence; the stores below depend on their
    // values, so no further system fence is needed here)
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const unsigned long long w = ((unsigned long long)(uint32_t)l[j] << 32) | (uint32_t)o[j];
        asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(&st->ctl.word[lane + 32 * j]), "l"(w) : "memory");
    }
    __syncwarp();
    __threadfence();
    if (lane == 0) {
        uint32_t g = atomicAdd(&st->ctl.gen, 1u) + 1u;
        if (st->clog_cap) {
            unsigned long long i = atomicAdd(&st->clog_count, 1ull);
            if (i < st->clog_cap) {
                ds_ctl_record r;
                r.ctl_gen = g;
                r.source = source;
                r.t = t0;
                st->clog[i] = r;
            }
        }
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------
// Loader warp (CTA 0): host mailbox -> HBM
// ---------------------------------------------------------------------------
__device__ void loader_loop(DevState* st) {
    const int lane = threadIdx.x & 31;
    HostMailbox* mb = st->mailbox;
    __shared__ uint32_t known_tail[DS_MAX_TENANTS];
    for (int i = lane; i < DS_MAX_TENANTS; i += 32) known_tail[i] = 0;
    __syncwarp();
    uint32_t last_gen = 0, last_pgen = 0, last_fgen = 0;
    uint64_t period = 0, next_flip = 0;
    int phase = 0;
    const uint64_t deadline = st->deadline_ns ? globaltimer() + st->deadline_ns : 0;
    const bool drain_exit = st->drain_exit != 0u;
    for (;;) {
        // one PCIe round trip per poll: lane i reads hot[4i .. 4i+3]
        uint4 hv;
        asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(hv.x), "=r"(hv.y), "=r"(hv.z), "=r"(hv.w)
                     : "l"(&mb->hot[4 * lane])
                     : "memory");
        // the compact control image (8 smids per lane), same round trip
        uint4 iv0, iv1;
        asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(iv0.x), "=r"(iv0.y), "=r"(iv0.z), "=r"(iv0.w)
                     : "l"(&mb->ctl_img[8 * lane])
                     : "memory");
        asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(iv1.x), "=r"(iv1.y), "=r"(iv1.z), "=r"(iv1.w)
                     : "l"(&mb->ctl_img[8 * lane + 4])
                     : "memory");
        const uint32_t ex = __shfl_sync(0xffffffffu, hv.y, 0);
        const uint32_t g = __shfl_sync(0xffffffffu, hv.x, 0);
        const uint32_t pg = __shfl_sync(0xffffffffu, hv.z, 0);
        const uint32_t fg = __shfl_sync(0xffffffffu, hv.w, 0);
        // acquire (system scope) only when the host published something: the
        // reads that follow (launch slots, control image, fault codes) must
        // not pass the poll; an idle poll skips the fence and comes round
        // sooner
        {
            bool tail_moved = false;
            if (lane >= kHotTail / 4 && lane < (kHotTail + DS_MAX_TENANTS) / 4) {
                const int t0 = 4 * lane - kHotTail;
                tail_moved = hv.x != known_tail[t0] || hv.y != known_tail[t0 + 1] || hv.z != known_tail[t0 + 2] ||
                             hv.w != known_tail[t0 + 3];
            }
            const bool changed = __any_sync(0xffffffffu, tail_moved) || g != last_gen || pg != last_pgen ||
                                 fg != last_fgen || ex != 0u;
            if (changed) asm volatile("fence.acq_rel.sys;" ::: "memory");
        }
        // a program enqueued before ds_start runs to completion and the
        // executor exits on its own (ds_set_drain_exit): usable when the host
        // cannot talk to a resident kernel, e.g. under a serialising profiler
        bool quit = ex != 0u || (deadline && globaltimer() >= deadline);
        quit = __shfl_sync(0xffffffffu, quit, 0);  // one decision for the whole warp
        if (drain_exit && !quit) {
            bool idle = true;
            for (int t = lane; t < DS_MAX_TENANTS; t += 32) {
                const uint32_t ht = ld_volatile_u32((const void*)&mb->hot[kHotTail + t]);
                const DevTenant* T = &st->tenants[t];
                idle &= ld_volatile_u32(&T->fault) != 0u ||
                        (known_tail[t] == ht && ld_acquire_u32(&T->head) == ht);
            }
            quit = __all_sync(0xffffffffu, idle);
        }
        if (quit) {
            if (lane == 0) {
                __threadfence();
                st_volatile_u32(&st->ctl.exit, 1u);
            }
            __syncwarp();
            return;
        }
        // new launches: tail of tenant t = hot[64 + t] -> lane 16 + t/4, component t%4
        for (int base = 0; base < DS_MAX_TENANTS; base += 32) {
            const int t = base + lane;
            const int src_lane = (kHotTail + t) >> 2, comp = t & 3;
            const uint32_t cx = __shfl_sync(0xffffffffu, hv.x, src_lane & 31);
            const uint32_t cy = __shfl_sync(0xffffffffu, hv.y, src_lane & 31);
            const uint32_t cz = __shfl_sync(0xffffffffu, hv.z, src_lane & 31);
            const uint32_t cw = __shfl_sync(0xffffffffu, hv.w, src_lane & 31);
            const uint32_t ht = comp == 0 ? cx : comp == 1 ? cy : comp == 2 ? cz : cw;
            const uint32_t kt = known_tail[t];
            unsigned pending = __ballot_sync(0xffffffffu, ht != kt);
            while (pending) {
                const int src = __ffs(pending) - 1;
                pending &= pending - 1;
                const int tt = base + src;
                const uint32_t from = __shfl_sync(0xffffffffu, kt, src);
                const uint32_t to = __shfl_sync(0xffffffffu, ht, src);
                // copy slots [from, to): lane l moves 16-B quarter (l & 3) of
                // slots s + (l >> 2) + 8k, k < 4 — 32 slots per batch with all
                // of a batch's PCIe reads in flight before any store (a decode
                // step enqueues ~160 slots at once)
                for (uint32_t s = from; s < to; s += 32) {
                    uint4 v[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t my = s + (lane >> 2) + 8 * k;
                        if (my < to) {
                            const uint32_t idx = (uint32_t)tt * (st->ring_mask + 1) + (my & st->ring_mask);
                            const uint4* hs = reinterpret_cast<const uint4*>(&st->host_rings[idx]) + (lane & 3);
                            asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                                         : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w)
                                         : "l"(hs)
                                         : "memory");
                        }
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t my = s + (lane >> 2) + 8 * k;
                        if (my < to) {
                            const uint32_t idx = (uint32_t)tt * (st->ring_mask + 1) + (my & st->ring_mask);
                            reinterpret_cast<uint4*>(&st->rings[idx])[lane & 3] = v[k];
                        }
                    }
                }
                __threadfence();  // every lane's slot stores before lane 0 publishes the tail
                __syncwarp();
                if (lane == 0) {
                    __threadfence();
                    st_release_u32(&st->tenants[tt].tail, to);
                    __threadfence();
                    try_open(st, tt);
                }
                __syncwarp();
                if (lane == src) known_tail[t] = to;
                __syncwarp();
            }
        }
        // injected local exceptions (ds_fault_inject): lane t/32 .. per tenant
        if (fg != last_fgen) {
            last_fgen = fg;
            asm volatile("fence.acq_rel.sys;" ::: "memory");
            for (int t = lane; t < DS_MAX_TENANTS; t += 32) {
                const uint32_t code = ld_volatile_u32((const void*)&mb->fault_req[t]);
                if (code && !ld_volatile_u32(&st->tenants[t].fault)) {
                    const uint32_t next = (uint32_t)(ld_volatile_u64(&st->tenants[t].claim) >> 32);
                    fault_tenant(st, t, code, next, 0xffffffffu);
                }
            }
            __syncwarp();
        }
        // control word: from the image read in this poll when every entry
        // carries the new generation's tag, else from the full arrays
        if (g != last_gen) {
            const uint32_t tag = g & 0xffffu;
            const uint32_t im[8] = {iv0.x, iv0.y, iv0.z, iv0.w, iv1.x, iv1.y, iv1.z, iv1.w};
            bool fresh = true;
#pragma unroll
            for (int k = 0; k < 8; ++k) fresh &= (im[k] >> 16) == tag;
            if (__all_sync(0xffffffffu, fresh)) {
                const uint64_t t0 = globaltimer();
                if (lane == 0) asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(&st->ctl.t_install), "l"(t0) : "memory");
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t e = im[k], ot = e & 0x7fu, lt = (e >> 7) & 0x7fu;
                    int32_t o = ot == kImgNone ? -1 : (int32_t)ot;
                    if (o >= 0) o |= ((e >> 14) & 1u ? kCtlSplit : 0) | ((e >> 15) & 1u ? kCtlOwnerOnly0 : 0);
                    const int32_t l = lt == kImgNone ? -1 : (int32_t)lt;
                    const unsigned long long w = ((unsigned long long)(uint32_t)l << 32) | (uint32_t)o;
                    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(&st->ctl.word[8 * lane + k]), "l"(w) : "memory");
                }
                __syncwarp();
                __threadfence();
                if (lane == 0) {
                    const uint32_t gg = atomicAdd(&st->ctl.gen, 1u) + 1u;
                    if (st->clog_cap) {
                        const unsigned long long i = atomicAdd(&st->clog_count, 1ull);
                        if (i < st->clog_cap) {
                            ds_ctl_record r;
                            r.ctl_gen = gg;
                            r.source = 0;
                            r.t = t0;
                            st->clog[i] = r;
                        }
                    }
                }
                __syncwarp();
            } else {
                install_ctl(st, (const int32_t*)mb->owner, (const int32_t*)mb->lender, true, 0, lane);
            }
            last_gen = g;
            // release (system scope): the installed words before the host sees the ack
            if (lane == 0) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(&mb->ack_gen), "r"(g) : "memory");
        }
        // periodic device-timer program (config 3 migration sweep): both
        // control words are copied into HBM once per program change, so a flip
        // is a device-local install
        if (pg != last_pgen) {
            last_pgen = pg;
            period = ld_acquire_sys_u64((const void*)&mb->periodic_ns);
            for (int k = 0; k < 2; ++k)
                for (int i = lane; i < DS_MAX_SMS; i += 32) {
                    st->per_owner[k][i] = (int32_t)ld_volatile_u32((const void*)&mb->per_owner[k][i]);
                    st->per_lender[k][i] = (int32_t)ld_volatile_u32((const void*)&mb->per_lender[k][i]);
                }
            __syncwarp();
            __threadfence();
            next_flip = globaltimer() + period;
            phase = 0;
        }
        if (period && globaltimer() >= next_flip) {
            phase ^= 1;
            install_ctl(st, st->per_owner[phase], st->per_lender[phase], false, 2, lane);
            next_flip += period;
        }
    }
}

// ---------------------------------------------------------------------------
// Scheduler warp (every CTA)
// ---------------------------------------------------------------------------
struct Claimed {
    int32_t tenant;
    uint32_t seq;
    uint32_t block;
    uint32_t grid;  // executed grid of the launch (known at claim: no re-read at retire)
    LaunchSlot* slot;
    bool retry;     // re-run of an abandoned block (from the retry ring)
    uint32_t resume;  // (spill slot + 1) | (k << 16) when it continues a spilled tile, else 0
};

// Per-scheduler memo of the launch it claimed from last: while that launch
// still had blocks, the next claim is a single atomicAdd (no pre-read).
struct ClaimCache {
    int32_t tenant = -1;
    uint32_t seq = 0;
    uint32_t grid = 0;
    bool more = false;
    LaunchSlot* slot = nullptr;
};

// Launch s is fully claimed: open s+1 for claims now (its blocks wait for s's
// completion before touching dependent data — wait_prev).  If s+1 is not
// enqueued yet, park the word closed; the loader opens it on publish
// (fence.sc on both sides, Dekker-style, so one of them does).
__device__ void open_next(DevState* st, int t, uint32_t s) {
    DevTenant* T = &st->tenants[t];
    const uint32_t nxt = s + 1;
    const uint32_t tail = ld_acquire_u32(&T->tail);
    if (nxt < tail) {
        atomicExch(&T->claim, ((unsigned long long)nxt << 32) | first_block(st, t, nxt));
        __threadfence();
        if (ld_volatile_u32(&T->fault)) kill_claim(T);
    } else {
        atomicExch(&T->claim, ((unsigned long long)nxt << 32) | kSat);
        __threadfence();
        try_open(st, t);
    }
}

__device__ bool try_claim(DevState* st, int t, Claimed& out, ClaimCache& cc) {
    DevTenant* T = &st->tenants[t];
    uint32_t s, grid;
    LaunchSlot* slot;
    if (!(cc.tenant == t && cc.more)) {
        unsigned long long w = ld_volatile_u64(&T->claim);
        s = (uint32_t)(w >> 32);
        uint32_t b = (uint32_t)w;
        if (b >= kSat) return false;
        if (cc.tenant == t && cc.seq == s) {
            slot = cc.slot;
            grid = cc.grid;
        } else {
            uint32_t tail = ld_acquire_u32(&T->tail);
            if (s >= tail) return false;
            slot = slot_of(st, t, s);
            grid = ld_volatile_u32(&slot->grid);
        }
        if (b >= grid) {
            cc.tenant = t;
            cc.seq = s;
            cc.grid = grid;
            cc.slot = slot;
            cc.more = false;
            return false;
        }
    } else {
        s = cc.seq;
        grid = cc.grid;
        slot = cc.slot;
    }
    unsigned long long old = atomicAdd(&T->claim, 1ull);
    uint32_t s2 = (uint32_t)(old >> 32), b2 = (uint32_t)old;
    if (b2 >= kSat) {
        cc.more = false;
        return false;
    }
    if (s2 != s) {
        // the word advanced since our read: the add landed on launch s2, which
        // is open (block field < kSat) hence enqueued
        slot = slot_of(st, t, s2);
        grid = ld_volatile_u32(&slot->grid);
    }
    cc.tenant = t;
    cc.seq = s2;
    cc.grid = grid;
    cc.slot = slot;
    if (b2 >= grid) {
        cc.more = false;
        return false;
    }
    cc.more = b2 + 1 < grid;
    // fully claimed: the next launch may start early — except for a tenant
    // whose blocks can be abandoned: its next launch opens at completion
    // (complete_launch), so no lane ever parks on launch s+1 while blocks of s
    // wait in the retry ring for a lane to run them
    if (b2 == grid - 1 && !((st->retry_mask >> t) & 1ull)) open_next(st, t, s2);
    out.tenant = t;
    out.seq = s2;
    out.block = b2;
    out.grid = grid;
    out.slot = slot;
    out.retry = false;
    out.resume = 0u;
    return true;
}

// ---- retry ring (abandoned blocks) ----
// Linear probing from the lane's home slot: concurrent pushers start apart,
// so a push is normally one CAS.  The occupancy bitmap after the slots is a
// hint for poppers (set after the entry is written, cleared after it is
// taken); the entries themselves are the truth.
__device__ void push_retry(DevState* st, int t, uint32_t seq, uint32_t block, int home) {
    const unsigned long long v = ((unsigned long long)(seq + 1) << 32) | block;
    unsigned long long* ring = st->retry + (size_t)t * kRetryStride;
    const int j = claim_retry_slot(ring, home, v, &st->ctl.exit);
    if (j < 0) return;  // exiting
    atomicOr(ring + kRetrySlots + (j >> 6), 1ull << (j & 63));
    __threadfence();  // entry (and hint) visible before the count says so
    atomicAdd(&st->tenants[t].retry_count, 1u);
}

__device__ __forceinline__ bool take_retry(DevState* st, int t, unsigned long long* ring, int j,
                                           unsigned long long v, Claimed& out) {
    const uint32_t k = ((uint32_t)v) >> kRetryBlockBits;
    // a spilled tile keeps its slot (TAKEN) until the resumer has read it back
    if (atomicCAS(ring + j, v, k ? kRetryTaken : 0ull) != v) return false;
    atomicAnd(ring + kRetrySlots + (j >> 6), ~(1ull << (j & 63)));
    atomicSub(&st->tenants[t].retry_count, 1u);
    out.tenant = t;
    out.seq = (uint32_t)(v >> 32) - 1u;
    out.block = (uint32_t)v & ((1u << kRetryBlockBits) - 1u);
    out.resume = k ? ((uint32_t)(j + 1) | (k << 16)) : 0u;
    out.slot = slot_of(st, t, out.seq);
    out.grid = ld_volatile_u32(&out.slot->grid);
    out.retry = true;
    return true;
}

// Oldest launch first (a later launch's blocks may be waiting for it); among
// its entries the one nearest the popper's home slot, so the lanes regaining
// SMs together do not all race for the same entry.  Fast path: up to 8
// occupied slots from the bitmap hint, nearest the home slot first; full
// scan when the hint shows none (a hint bit can lag a racing push).
__device__ bool try_retry(DevState* st, int t, Claimed& out, int home) {
    if (!((st->retry_mask >> t) & 1ull)) return false;
    DevTenant* T = &st->tenants[t];
    if (ld_volatile_u32(&T->retry_count) == 0u) return false;
    // a failed tenant's abandoned blocks are never re-run (its launches never complete)
    if (ld_volatile_u32(&T->fault) != 0u) return false;
    unsigned long long* ring = st->retry + (size_t)t * kRetryStride;
    constexpr int kWords = (kRetrySlots + 63) / 64;
    for (int attempt = 0; attempt < 8; ++attempt) {
        unsigned long long bm[kWords];
#pragma unroll
        for (int w = 0; w < kWords; ++w) bm[w] = ld_volatile_u64(ring + kRetrySlots + w);
        int cand[8], nc = 0;
        for (int ww = 0; ww <= kWords && nc < 8; ++ww) {
            const int w = (home / 64 + ww) % kWords;
            unsigned long long b = bm[w];
            if (ww == 0) b &= ~0ull << (home & 63);            // from the home slot on ...
            else if (ww == kWords) b = bm[w] & ((1ull << (home & 63)) - 1ull);  // ... wrapping to it
            while (b && nc < 8) {
                const int bit = __ffsll((long long)b) - 1;
                b &= b - 1;
                cand[nc++] = w * 64 + bit;
            }
        }
        if (nc == 0) break;
        unsigned long long v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = k < nc ? ld_volatile_u64(ring + cand[k]) : 0ull;
        int bk = -1;
        uint32_t best = ~0u;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (v[k] > kRetryTaken && (uint32_t)(v[k] >> 32) < best) {
                best = (uint32_t)(v[k] >> 32);
                bk = k;
            }
        if (bk < 0) break;
        if (take_retry(st, t, ring, cand[bk], v[bk], out)) return true;
    }
    // full scan (hint empty or stale)
    for (int attempt = 0; attempt < 8; ++attempt) {
        uint32_t best_seq = ~0u;
        int bj = -1, bd = kRetrySlots;
        unsigned long long bv = 0ull;
        // 16-B loads, all issued before the compares consume them
#pragma unroll 32
        for (int j = 0; j < kRetrySlots; j += 2) {
            unsigned long long x[2];
            asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(x[0]), "=l"(x[1]) : "l"(ring + j) : "memory");
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                if (x[e] <= kRetryTaken) continue;  // free, or a spill being written / read
                const uint32_t sq = (uint32_t)(x[e] >> 32);
                const int d = (j + e - home + kRetrySlots) % kRetrySlots;
                if (sq < best_seq || (sq == best_seq && d < bd)) {
                    best_seq = sq;
                    bd = d;
                    bj = j + e;
                    bv = x[e];
                }
            }
        }
        if (bj < 0) return false;
        if (take_retry(st, t, ring, bj, bv, out)) return true;
    }
    return false;
}

__device__ void complete_launch(DevState* st, int t, uint32_t seq, LaunchSlot* slot) {
    DevTenant* T = &st->tenants[t];
    // ordered after every block's writes by the acq_rel retire atomic
    const uint64_t tend = globaltimer();
    // 1. publish completion first (critical path: early-started blocks of the
    //    next launch are waiting on head); the streamed word moves to the next
    //    launch before, so its blocks' marks (made after they see head) count
    *reinterpret_cast<volatile unsigned long long*>(&T->streamed) = (unsigned long long)(seq + 1) << 32;
    st_release_u32(&T->head, seq + 1);
    // abandonable tenants open their next launch only now (see try_claim)
    if ((st->retry_mask >> t) & 1ull) open_next(st, t, seq);
    // 2. device -> host completion record (PCIe, off the critical path)
    unsigned long long i = atomicAdd(&st->completion_count, 1ull);
    HostCompletion* hc = &st->completions[i & st->completion_mask];
    ds_completion c;
    c.tenant = t;
    c.kernel = ld_volatile_u32(&slot->kernel_id);
    c.seq = seq;
    c.launch_tag = ld_volatile_u64(&slot->tag);
    c.grid = ld_volatile_u32(&slot->grid);
    c.sms_used = ld_volatile_u32(&slot->sms);
    c.t_first_claim = ld_volatile_u64(&slot->t_first);
    c.t_end = tend;
    hc->c = c;
    __threadfence_system();
    st_release_sys_u64((void*)&hc->valid, i + 1);
}

__device__ void maybe_fire_trigger(DevState* st, const Claimed& w, int lane) {
    uint32_t k = 0;
    if (lane == 0) k = ld_volatile_u32(&st->trig_next);
    k = __shfl_sync(0xffffffffu, k, 0);
    if (k >= ld_volatile_u32(&st->trig_count)) return;
    const ClaimTrigger* tr = &st->triggers[k];
    bool fire = false;
    if (lane == 0) {
        if (tr->tenant == w.tenant && tr->seq == w.seq && w.block >= tr->block) {
            fire = atomicCAS(&st->trig_next, k, k + 1) == k;
        }
    }
    fire = __shfl_sync(0xffffffffu, fire, 0);
    if (fire) install_ctl(st, tr->owner, tr->lender, false, 1, lane);
}

// A lane leaves tenant t (switch or idle): if its SM no longer serves t, the
// control change revoked it — the block it was running when the change came
// is the boundary wait (install -> that block's retire).
__device__ __forceinline__ void ledger_leave(DevState* st, unsigned long long cw, int32_t t, uint64_t t_last_retire) {
    if (serves_tenant(cw, t)) return;
    const uint64_t t_ins = ld_volatile_u64(&st->ctl.t_install);
    atomicAdd(&st->led_yields, 1ull);
    if (t_last_retire > t_ins) atomicAdd(&st->led_yield_ns, (unsigned long long)(t_last_retire - t_ins));
}

__device__ void scheduler_loop(DevState* st, Stage* stage, volatile uint64_t* body_t0, volatile uint32_t* ab_flag,
                               volatile uint32_t* ab_info, uint32_t sm, int lane_id) {
    const int kFull = bar_full(lane_id), kEmpty = bar_empty(lane_id), kDone = bar_done(lane_id);
    const int lane = threadIdx.x & 31;
    int32_t last_tenant = -1;
    uint32_t last_seq = 0xffffffffu;
    const int home = (int)(sm * kLanes + lane_id) % kRetrySlots;  // this lane's retry-ring slot
    bool idle_logged = false;
    uint64_t t_last_retire = 0, t_last_switch = 0;  // ledger (lane 0 of the warp)
    uint32_t backoff = 32;
    bool have_prev = false;
    Claimed prev{};
    ClaimCache cc;
    for (;;) {
        // ---- retire the block the body just finished ----
        if (have_prev) {
            named_sync(kDone, kBodyThreads + 32);
            const bool abandoned = *ab_flag != 0u;  // written by the body before kDone
            if (lane == 0 && abandoned) {
                // the block gave up (revoked SM / waiting on abandoned work):
                // it re-runs from scratch on the next claimer, never retires here
                *ab_flag = 0u;
                const uint32_t info = *ab_info;
                *ab_info = 0u;
                if (info) {
                    // the body spilled its accumulators into slot j (reserved):
                    // publish the entry there, continuing at k-block k
                    const int j = (int)(info & 0xffffu) - 1;
                    const uint32_t k = info >> 16;
                    unsigned long long* ring = st->retry + (size_t)prev.tenant * kRetryStride;
                    __threadfence();  // the spill (ordered by kDone) before the entry
                    atomicExch(ring + j, ((unsigned long long)(prev.seq + 1) << 32) |
                                             ((unsigned long long)k << kRetryBlockBits) | prev.block);
                    atomicOr(ring + kRetrySlots + (j >> 6), 1ull << (j & 63));
                    __threadfence();
                    atomicAdd(&st->tenants[prev.tenant].retry_count, 1u);
                } else {
                    push_retry(st, prev.tenant, prev.seq, prev.block, home);
                }
                t_last_retire = globaltimer();
                if (st->blog_cap) {
                    unsigned long long i = atomicAdd(&st->blog_count, 1ull);
                    if (i < st->blog_cap) {
                        ds_block_record br;
                        br.tenant = prev.tenant;
                        br.seq = prev.seq;
                        br.block = prev.block;
                        br.smid = (uint16_t)sm;
                        br.flags = 1;  // abandoned attempt: t_start = when it decided to stop
                        br.t_start = *tc_stop_time_of(lane_id);
                        br.t_end = globaltimer();
                        st->blog[i] = br;
                    }
                }
            } else if (lane == 0) {
                uint64_t t1 = globaltimer();
                t_last_retire = t1;
                uint64_t t0 = *body_t0;
                // release: the body's writes (ordered before this thread by the
                // kDone barrier, cumulativity) are published with the retire;
                // acquire: the completer sees every other block's writes
                uint32_t r;
                asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(r) : "l"(&prev.slot->retired) : "memory");
                atomicAdd(&st->blocks_executed, 1ull);
                if (st->blog_cap) {
                    unsigned long long i = atomicAdd(&st->blog_count, 1ull);
                    if (i < st->blog_cap) {
                        ds_block_record br;
                        br.tenant = prev.tenant;
                        br.seq = prev.seq;
                        br.block = prev.block;
                        br.smid = (uint16_t)sm;
                        br.flags = 0;
                        br.t_start = t0;
                        br.t_end = t1;
                        st->blog[i] = br;
                    }
                }
                if (r == prev.grid - 1) complete_launch(st, prev.tenant, prev.seq, prev.slot);
            }
            __syncwarp();
            have_prev = false;
        }
        // ---- claim the next block for this SM ----
        Claimed w{};
        bool got = false, exit_now = false;
        if (lane == 0) {
            unsigned long long cw = ~0ull;
            for (;;) {
                // both words requested before either is used: one L2 round trip
                const uint32_t ex = ld_volatile_u32(&st->ctl.exit);
                // the SM's own control word, by %smid read at the boundary
                // (a resident CTA never changes SM, so this equals the value
                // read at start; reading it here keeps the arbiter's contract
                // "each boundary consults the word of the SM it runs on")
                cw = ld_volatile_u64(&st->ctl.word[smid()]);
                if (ex) { exit_now = true; break; }
                int32_t ow = (int32_t)(uint32_t)cw;
                const int32_t ln = (int32_t)(uint32_t)(cw >> 32);
                int32_t first = ow, second = ln;
                if (ow >= 0) {
                    ow &= kCtlTenantMask;
                    first = ow;
                    const int32_t f = (int32_t)(uint32_t)cw;
                    if ((f & kCtlSplit) && lane_id == 1) {
                        first = ln;
                        second = ow;
                    } else if ((f & kCtlOwnerOnly0) && lane_id == 0) {
                        second = -1;
                    }
                }
                if (first >= 0 && first < DS_MAX_TENANTS &&
                    (try_retry(st, first, w, home) || try_claim(st, first, w, cc))) {
                    got = true;
                    break;
                }
                if (second >= 0 && second < DS_MAX_TENANTS && second != first &&
                    (try_retry(st, second, w, home) || try_claim(st, second, w, cc))) {
                    got = true;
                    break;
                }
                if (!idle_logged && last_tenant != -1) ledger_leave(st, cw, last_tenant, t_last_retire);
                if (!idle_logged && last_tenant != -1 && st->slog_cap) {
                    unsigned long long i = atomicAdd(&st->slog_count, 1ull);
                    if (i < st->slog_cap) {
                        ds_switch_record r;
                        r.smid = (uint16_t)sm;
                        r.from_tenant = (int16_t)last_tenant;
                        r.to_tenant = -1;
                        r.pad = 0;
                        r.ctl_gen = ld_volatile_u32(&st->ctl.gen);
                        r.t = globaltimer();
                        st->slog[i] = r;
                    }
                    idle_logged = true;
                }
                if (last_tenant != -1) {
                    idle_logged = true;
                    last_tenant = -1;
                }
                __nanosleep(backoff);
                if (backoff < 256) backoff <<= 1;
            }
            if (got) {
                backoff = 32;
                if (w.tenant != last_tenant) {
                    const uint64_t now = globaltimer();
                    if (last_tenant >= 0) {
                        ledger_leave(st, cw, last_tenant, t_last_retire);
                        atomicAdd(&st->led_switches, 1ull);
                        atomicAdd(&st->led_switch_ns, (unsigned long long)(now - t_last_retire));
                    }
                    const uint64_t t_ins = ld_volatile_u64(&st->ctl.t_install);
                    if (t_ins > t_last_switch && now > t_ins) {  // moved here by a control change
                        atomicAdd(&st->led_grants, 1ull);
                        atomicAdd(&st->led_grant_ns, (unsigned long long)(now - t_ins));
                    }
                    t_last_switch = now;
                }
                // no fence here: bodies acquire earlier launches' results in wait_prev
                // the slot's first 32 B (body, grid, gx, gy, gz, kernel_id, args)
                // in two vector loads issued together: one L2 round trip
                uint4 h0, h1;
                asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(h0.x), "=r"(h0.y), "=r"(h0.z), "=r"(h0.w) : "l"(w.slot) : "memory");
                asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(h1.x), "=r"(h1.y), "=r"(h1.z), "=r"(h1.w)
                             : "l"(reinterpret_cast<const char*>(w.slot) + 16) : "memory");
                Stage s;
                s.tenant = w.tenant;
                s.body = (int32_t)h0.x;
                s.seq = w.seq;
                s.block = w.block;
                s.gx = h0.z;
                s.gy = h0.w;
                s.gz = h1.x;
                s.pad = w.resume;
                s.args = ((uint64_t)h1.w << 32) | h1.z;
                *stage = s;
            } else {
                stage->tenant = -1;
            }
        }
        __syncwarp();
        named_arrive(kFull, kBodyThreads + 32);
        exit_now = __shfl_sync(0xffffffffu, exit_now, 0);
        got = __shfl_sync(0xffffffffu, got, 0);
        if (!got) {  // exit: let the body warps read the exit stage, then leave
            named_sync(kEmpty, kBodyThreads + 32);
            break;
        }
        w.tenant = __shfl_sync(0xffffffffu, w.tenant, 0);
        w.seq = __shfl_sync(0xffffffffu, w.seq, 0);
        w.block = __shfl_sync(0xffffffffu, w.block, 0);
        w.slot = (LaunchSlot*)__shfl_sync(0xffffffffu, (unsigned long long)w.slot, 0);
        w.grid = __shfl_sync(0xffffffffu, w.grid, 0);
        // ---- bookkeeping while the body runs ----
        if (lane == 0) {
            if (w.block == 0 && !w.retry) w.slot->t_first = globaltimer();
            if (w.tenant != last_tenant || w.seq != last_seq) {
                atomicAdd(&w.slot->sms, 1u);
                if (w.tenant != last_tenant && st->slog_cap) {
                    unsigned long long i = atomicAdd(&st->slog_count, 1ull);
                    if (i < st->slog_cap) {
                        ds_switch_record r;
                        r.smid = (uint16_t)sm;
                        r.from_tenant = (int16_t)last_tenant;
                        r.to_tenant = (int16_t)w.tenant;
                        r.pad = 0;
                        r.ctl_gen = ld_volatile_u32(&st->ctl.gen);
                        r.t = globaltimer();
                        st->slog[i] = r;
                    }
                }
            }
            last_tenant = w.tenant;
            last_seq = w.seq;
            idle_logged = false;
        }
        __syncwarp();
        maybe_fire_trigger(st, w, lane);
        named_sync(kEmpty, kBodyThreads + 32);  // body copied the stage
        prev = w;
        have_prev = true;
    }
}

// ---------------------------------------------------------------------------
// Body warps
// ---------------------------------------------------------------------------
__device__ void body_loop(DevState* st, Stage* stage, volatile uint64_t* body_t0, volatile uint32_t* ab_flag,
                          volatile uint32_t* ab_info, char* smem, uint32_t smem_bytes, uint32_t tmem_base, int lane_id) {
    auto prev_head_of = [&](int t) { return &st->tenants[t].head; };
    const int kFull = bar_full(lane_id), kEmpty = bar_empty(lane_id), kDone = bar_done(lane_id);
    for (;;) {
        named_sync(kFull, kBodyThreads + 32);
        Stage s = *stage;
        named_arrive(kEmpty, kBodyThreads + 32);
        if (s.tenant < 0) return;
        if (ltid() == 0) *body_t0 = globaltimer();
        BodyCtx c;
        c.gx = s.gx;
        c.gy = s.gy;
        c.gz = s.gz;
        c.bx = s.block % s.gx;
        c.by = (s.block / s.gx) % s.gy;
        c.bz = s.block / (s.gx * s.gy);
        c.args = reinterpret_cast<const void*>(s.args);
        c.smem = smem;
        c.smem_bytes = smem_bytes;
        c.tmem_base = tmem_base;
        c.prev_head = prev_head_of(s.tenant);
        c.seq = s.seq;
        c.dbg = nullptr;
        c.st = st;
        c.tenant = s.tenant;
        c.abandon = ((st->retry_mask >> s.tenant) & 1ull) ? ab_flag : nullptr;
        c.ab_info = ab_info;
        c.resume = s.pad;
        run_body(s.body, c);
        // the scheduler's release (acq_rel retire atomic after this barrier)
        // publishes this thread's writes at gpu scope
        named_arrive(kDone, kBodyThreads + 32);
    }
}

extern "C" __global__ void __launch_bounds__(kExecThreads, 1) ds_executor_kernel(DevState* st, uint32_t smem_bytes) {
    extern __shared__ __align__(1024) char smem[];
    __shared__ Stage stage[kLanes];
    __shared__ volatile uint64_t body_t0[kLanes];
    __shared__ volatile uint32_t ab_flag[kLanes];
    __shared__ volatile uint32_t ab_info[kLanes];
    const int warp = threadIdx.x >> 5;
    const uint32_t sm = smid();
    if (warp == kLoaderWarp) {
        if (blockIdx.x == 0) loader_loop(st);
        return;
    }
    // TMEM: one allocation for the CTA's lifetime, split between the lanes
    __shared__ uint32_t tmem_base_sh;
    if (warp == 0) tc::tmem_alloc(&tmem_base_sh, kTmemCols);
    if (threadIdx.x < kLanes) {  // ordered by the barrier below
        ab_flag[threadIdx.x] = 0u;
        ab_info[threadIdx.x] = 0u;
        g_desc_fenced[threadIdx.x] = nullptr;
    }
    tc::tc_fence_before();
    named_sync(kBarExit, kLanes * (kBodyThreads + 32));
    tc::tc_fence_after();
    const uint32_t lane_smem = smem_bytes / kLanes;
    if (warp >= kSchedWarp0) {
        const int l = warp - kSchedWarp0;
        scheduler_loop(st, &stage[l], &body_t0[l], &ab_flag[l], &ab_info[l], sm, l);
    } else {
        const int l = warp >> 3;
        body_loop(st, &stage[l], &body_t0[l], &ab_flag[l], &ab_info[l], smem + l * lane_smem, lane_smem,
                  tmem_base_sh + l * kLaneTmemCols, l);
    }
    tc::tc_fence_before();
    named_sync(kBarExit, kLanes * (kBodyThreads + 32));
    tc::tc_fence_after();
    if (warp == 0) tc::tmem_dealloc(tmem_base_sh, kTmemCols);
}

// Solo baseline: the same body as a plain grid (exclusive_baseline,
// src/engine/engine.cpp:1400-1417).  256 threads, blockIdx = logical block.
// optional per-CTA stamps of the solo wrapper (ds_solo_trace): entry, TMEM
// allocated, body returned, exit -- where a plain-grid launch spends time
// outside the body
__device__ unsigned long long* g_solo_trace = nullptr;

extern "C" __global__ void __launch_bounds__(kBodyThreads, 1)
    ds_solo_kernel(int body, const void* args, uint32_t gx, uint32_t gy, uint32_t gz, uint32_t smem_bytes) {
    extern __shared__ __align__(1024) char smem[];
    uint32_t b = blockIdx.x;
    unsigned long long* const tr = g_solo_trace;
    if (tr && threadIdx.x == 0) tr[(size_t)b * 4] = globaltimer();
    BodyCtx c;
    c.gx = gx;
    c.gy = gy;
    c.gz = gz;
    c.bx = b % gx;
    c.by = (b / gx) % gy;
    c.bz = b / (gx * gy);
    c.args = args;
    c.smem = smem;
    c.smem_bytes = smem_bytes;
    c.prev_head = nullptr;
    c.seq = 0;
    c.dbg = nullptr;
    c.st = nullptr;
    c.tenant = -1;
    c.abandon = nullptr;
    c.ab_info = nullptr;
    c.resume = 0u;
    __shared__ uint32_t tmem_base_sh;
    const bool tc_body = body == DS_BODY_GEMM_BF16 || body == DS_BODY_GEMV_BF16 || body == DS_BODY_ATTN_DECODE;
    if (tc_body) {
        if ((threadIdx.x >> 5) == 0) tc::tmem_alloc(&tmem_base_sh, kLaneTmemCols);
        tc::tc_fence_before();
        __syncthreads();
        tc::tc_fence_after();
        c.tmem_base = tmem_base_sh;
    } else {
        c.tmem_base = 0;
    }
    if (tr && threadIdx.x == 0) tr[(size_t)b * 4 + 1] = globaltimer();
    run_body(body, c);
    if (tr && threadIdx.x == 0) tr[(size_t)b * 4 + 2] = globaltimer();
    if (tc_body) {
        tc::tc_fence_before();
        __syncthreads();
        tc::tc_fence_after();
        if ((threadIdx.x >> 5) == 0) tc::tmem_dealloc(c.tmem_base, kLaneTmemCols);
    }
    if (tr && threadIdx.x == 0) tr[(size_t)b * 4 + 3] = globaltimer();
}

extern "C" __global__ void ds_probe_kernel(uint32_t* smids, uint32_t* nsmid, uint64_t* timer) {
    if (threadIdx.x == 0) {
        smids[blockIdx.x] = smid();
        uint32_t n;
        asm volatile("mov.u32 %0, %%nsmid;" : "=r"(n));
        if (blockIdx.x == 0) {
            *nsmid = n;
            *timer = globaltimer();
        }
    }
}

}  // namespace ds

// host-side launch shims (called from runtime.cpp)
static cudaError_t exec_attrs(uint32_t smem) {
    cudaError_t e = cudaFuncSetAttribute(ds::ds_executor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // all of the unified L1/shared array as shared memory: the worker CTAs of
    // one SM must fit side by side
    return cudaFuncSetAttribute(ds::ds_executor_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                (int)cudaSharedmemCarveoutMaxShared);
}

extern "C" cudaError_t ds_dev_launch_executor(ds::DevState* st, int num_ctas, uint32_t smem, cudaStream_t s) {
    cudaError_t e = exec_attrs(smem);
    if (e != cudaSuccess) return e;
    void* args[] = {&st, &smem};
    return cudaLaunchCooperativeKernel((void*)ds::ds_executor_kernel, dim3(num_ctas), dim3(ds::kExecThreads), args,
                                       smem, s);
}

extern "C" cudaError_t ds_dev_executor_occupancy(uint32_t smem, int* blocks_per_sm) {
    cudaError_t e = exec_attrs(smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, ds::ds_executor_kernel, ds::kExecThreads, smem);
}

extern "C" cudaError_t ds_dev_solo_trace(void* buf) {
    unsigned long long* p = reinterpret_cast<unsigned long long*>(buf);
    return cudaMemcpyToSymbol(ds::g_solo_trace, &p, sizeof(p));
}

extern "C" cudaError_t ds_dev_launch_solo(int body, const void* args, uint32_t gx, uint32_t gy, uint32_t gz,
                                          uint32_t smem, cudaStream_t s) {
    // attributes set once per size (and the carveout pinned to max shared, the
    // configuration every tensor-core body needs), not per launch
    // per device (function attributes are per device context); concurrent
    // launchers at worst both set the same attributes
    static std::atomic<int> cur_smem[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        dev = 0;
        cur_smem[0].store(0);
    }
    const int have = cur_smem[dev].load(std::memory_order_relaxed);
    if ((int)smem > have || have == 0) {
        cudaError_t e = cudaFuncSetAttribute(ds::ds_solo_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(ds::ds_solo_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 (int)cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        cur_smem[dev].store((int)smem, std::memory_order_relaxed);
    }
    ds::ds_solo_kernel<<<dim3(gx * gy * gz), dim3(ds::kBodyThreads), smem, s>>>(body, args, gx, gy, gz, smem);
    return cudaGetLastError();
}

// fp32 FFMA throughput probe (config 1's roofline denominator): 8
// independent fma chains per thread, 4 blocks x 256 threads per SM; the
// result is kept live so nothing is folded away
extern "C" __global__ void __launch_bounds__(256) ds_ffma_probe_kernel(float* out, int iters, float x) {
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = x + (float)(threadIdx.x + j);
    const float b = 1.0000001f, c = 1e-7f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = __fmaf_rn(a[j], b, c);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j];
    if (s == 12345.678f) out[blockIdx.x] = s;
}

extern "C" cudaError_t ds_dev_ffma_probe(int nblocks, int iters, float* out, cudaStream_t s) {
    ds_ffma_probe_kernel<<<nblocks, 256, 0, s>>>(out, iters, 1.f);
    return cudaGetLastError();
}

extern "C" cudaError_t ds_dev_probe(int nblocks, uint32_t* smids, uint32_t* nsmid, uint64_t* timer, cudaStream_t s) {
    ds::ds_probe_kernel<<<nblocks, 32, 0, s>>>(smids, nsmid, timer);
    return cudaGetLastError();
}

extern "C" uint32_t ds_dev_body_smem(int body) {
    switch (body) {
        case DS_BODY_REDUCE_CHUNKS: return 16384 * 4 + 1024;
        case DS_BODY_SGEMM: return (64 * ds::kSgA + 32 * 64) * 4 + 1024;
        case DS_BODY_SPIN: return 1024;
        case DS_BODY_GEMM_BF16: return ds::TcSmem<ds::kGemmBN, ds::kGemmStages>::kBytes + 1024;
        case DS_BODY_GEMV_BF16: {
            const uint32_t a = ds::TcSmem<ds::kGemvBN, ds::kGemvStages>::kBytes;
            const uint32_t b = ds::TcSmem<ds::kGemvBN, ds::kGemvStages64, ds::kTcBK, 64>::kBytes;
            return (a > b ? a : b) + 1024;
        }
        case DS_BODY_ATTN_DECODE: return (ds::kAttnSmem > ds::kAtSmem ? ds::kAttnSmem : ds::kAtSmem) + 1024;
        case DS_BODY_RMSNORM: return 1024;
        case DS_BODY_EMBED: return 1024;
        case DS_BODY_ARGMAX: return 1024;
        case DS_BODY_SPLITK_REDUCE: return 1024;
        case DS_BODY_ALLREDUCE_P2P: return 1024;
        case DS_BODY_CHECKSUM: return 1024;
        default: return ds::kDefaultSmem;
    }
}

extern "C" int ds_attn_chunk(void) { return ds::kAttnChunk; }

extern "C" int ds_dev_ctas_per_sm(void) { return 1; }  // one CTA per SM (kLanes worker lanes inside)

extern "C" int ds_dev_exec_attrs(int* regs, int* local, int* static_smem, int* max_threads) {
    cudaFuncAttributes a;
    if (cudaFuncGetAttributes(&a, ds::ds_executor_kernel) != cudaSuccess) return -1;
    *regs = a.numRegs;
    *local = (int)a.localSizeBytes;
    *static_smem = (int)a.sharedSizeBytes;
    *max_threads = a.maxThreadsPerBlock;
    return 0;
}
