// Shared host/device layout of the GPU-coroutine runtime.
//
// HBM layout (one domain = one GPU):
//   DevState            control words, per-tenant claim words, counters, log cursors
//   rings[64][R]        launch slots (64 B each), program order per tenant
//   args arena          immutable kernel argument blocks (512 B each)
//   block/switch/ctl logs
// Host-mapped pinned memory:
//   HostMailbox         host -> device: tails, control word, exit, periodic program
//   host rings[64][R]   host -> device launch slots (copied into HBM by the loader warp)
//   completion ring     device -> host: ds_completion records
#pragma once

#include <stdint.h>

#include "../../include/detshare/ds.h"

namespace ds {

#ifndef DS_LANES
#define DS_LANES 2
#endif
// Worker lanes per executor CTA (one CTA per SM).  Each lane = 8 body warps +
// 1 scheduler warp with its own barriers, smem half and TMEM columns; two
// lanes let one stream a block while the other claims / fills its pipeline.
constexpr int kLanes = DS_LANES;
constexpr int kCtasPerSm = kLanes;  // tile/pipeline sizing follows the number of concurrent workers per SM
constexpr uint32_t kSat = 0x40000000u;      // claim-word block field >= kSat: kernel not open
constexpr uint32_t kDead = 0x80000000u;     // claim-word block field of a failed tenant (never reopens)
constexpr int kBodyThreads = 256;           // warps 8L..8L+7 run lane L's tenant bodies
constexpr int kSchedWarp0 = 8 * kLanes;     // scheduler warp of lane L = kSchedWarp0 + L
constexpr int kLoaderWarp = 9 * kLanes;     // CTA 0 only: host mailbox poller
constexpr int kExecThreads = 32 * (9 * kLanes + 1);
constexpr int kMaxArgs = 512;
constexpr uint32_t kLaneSmem = kLanes == 2 ? 104 * 1024 : 200 * 1024;  // dynamic smem per lane
constexpr uint32_t kDefaultSmem = kLaneSmem * kLanes;
constexpr int kMaxTriggers = 64;
// Retry ring per tenant: blocks abandoned mid-way (an abandonable body whose
// SM was revoked, or that waited on a launch with abandoned blocks) are
// re-run from scratch by the next claimer.  Entry = ((seq + 1) << 32) | block.
constexpr int kRetrySlots = 320;  // >= worker lanes (2 x 148): a lane holds at most one entry of its own
constexpr int kRetryStride = kRetrySlots + 8;  // per tenant: the slots, then an occupancy bitmap (5 words, a hint)
// Ring entry values: 0 free, kRetryReserved (a spill in progress), kRetryTaken
// (a resumer is reading the spill), else ((seq + 1) << 32) | (k << 20) | block
// with k the next k-block of a spilled tile (0: restart from scratch).
constexpr unsigned long long kRetryReserved = 1ull, kRetryTaken = 2ull;
constexpr uint32_t kRetryBlockBits = 20;
constexpr int kSaveFloats = 128 * 256;  // one spilled 128 x 256 fp32 accumulator tile
// GemmArgs fields the host validates for abandonable GEMMs (entry encoding:
// block < 2^20, k-block < 2^12); asserted against the struct in gemm_tc.cuh
constexpr size_t kGemmArgsOffK = 272, kGemmArgsOffBk = 296, kGemmArgsOffAbandon = 304;
constexpr size_t kGemmArgsBody = 448;

// Named barrier ids (0 reserved).  Lane 0: body 1, full 2, empty 3, done 4,
// epilogue 7; lane 1: body 8, full 9, empty 10, done 11, epilogue 12; 5 = exit.
__host__ __device__ constexpr int bar_full(int lane) { return lane ? 9 : 2; }
__host__ __device__ constexpr int bar_empty(int lane) { return lane ? 10 : 3; }
__host__ __device__ constexpr int bar_done(int lane) { return lane ? 11 : 4; }
constexpr int kBarExit = 5;

struct alignas(64) LaunchSlot {
    int32_t body;
    uint32_t grid;       // executed logical grid size (gx*gy*gz)
    uint32_t gx, gy, gz;
    int32_t kernel_id;
    uint64_t args;       // device pointer into the args arena
    uint64_t tag;
    uint32_t retired;    // device: retired blocks
    uint32_t sms;        // device: distinct SMs that ran this launch
    uint64_t t_first;    // device: first claim time
    uint32_t seq;        // low 32 bits of the launch sequence
    uint32_t flags;
};
static_assert(sizeof(LaunchSlot) == 64, "slot is one 64-byte line");

struct alignas(128) DevTenant {
    unsigned long long claim;  // (seq << 32) | next_block ; block >= kSat => not open
    uint32_t tail;             // launches visible to the device
    uint32_t head;             // launches completed
    unsigned long long blocks; // blocks executed (stats)
    uint32_t fault;            // local-exception code, 0 = healthy (set once, never cleared)
    uint32_t retry_count;      // abandoned blocks waiting in the tenant's retry ring
    uint32_t save_base;        // first spill slot of this tenant in DevState::save (abandonable tenants)
    uint32_t pad0;
    // (seq << 32) | blocks of launch seq whose HBM streaming is done
    // (mark_streamed): the next launch's early-started blocks prefetch into L2
    // once the whole launch has streamed, i.e. while its epilogues run
    unsigned long long streamed;
    uint32_t pad[20];
};
static_assert(sizeof(DevTenant) == 128, "tenant word owns a 128-byte line");

struct ClaimTrigger {
    int32_t tenant;
    uint32_t seq;
    uint32_t block;
    uint32_t pad;
    int32_t owner[DS_MAX_SMS];   // by smid
    int32_t lender[DS_MAX_SMS];
};

// Owner-field flags of a control word (owner >= 0 only): lane split — the
// SM's two worker lanes serve different tenants.  Lane 1 claims the lender
// first (then the owner); with kCtlOwnerOnly0, lane 0 never runs the lender.
// A memory-bound owner and a compute-bound lender then share every SM.
constexpr int32_t kCtlSplit = 1 << 30;
constexpr int32_t kCtlOwnerOnly0 = 1 << 29;
constexpr int32_t kCtlTenantMask = 0xffff;

struct alignas(128) DevControl {
    unsigned long long word[DS_MAX_SMS];  // by physical smid: (lender << 32) | owner, -1 = none
    uint32_t gen;                // bumped on every control change (any source)
    uint32_t exit;
    unsigned long long t_install;  // %globaltimer when the current control word started installing
    uint32_t pad[28];
};

struct HostCompletion {
    ds_completion c;
    volatile unsigned long long valid;  // index + 1 once c is written
    unsigned long long pad;
};
static_assert(sizeof(HostCompletion) == 64, "completion record is one line");

// Device -> host record of a tenant's local exception (written once; `code`
// last, with release).
struct HostFault {
    volatile uint32_t code;
    volatile uint32_t seq;    // launch that was running (raise) or next to claim (injection)
    volatile uint32_t block;  // logical block that raised (0xffffffff: injected)
    volatile uint32_t head;   // launches completed when it faulted (= first failed launch)
    volatile unsigned long long t;  // %globaltimer ns
    unsigned long long pad2;
};
static_assert(sizeof(HostFault) == 32, "fault record");

// Host -> device mailbox.  Everything the loader polls sits in one 512-B
// "hot" block read with a single warp-wide 16-B/lane load per poll:
//   hot[0] control generation, hot[1] exit, hot[2] periodic-program generation,
//   hot[3] fault-request generation, hot[64 + t] launch tail of tenant t.
// Compact control image, polled in the same PCIe round trip as hot[]: one
// 32-bit entry per smid = owner (7 bits, 0x7f none) | lender << 7 (7 bits)
// | split << 14 | owner-only-lane-0 << 15 | generation tag << 16.  The
// loader installs it from the poll that announced the generation when every
// entry carries that generation's tag (32-bit host stores are atomic), so a
// control change costs no second round trip; a torn read waits one poll.
constexpr uint32_t kImgNone = 0x7fu;
struct HostMailbox {
    volatile uint32_t hot[128];
    volatile uint32_t ctl_img[DS_MAX_SMS];
    volatile unsigned long long periodic_ns;
    volatile int32_t owner[DS_MAX_SMS];   // by smid
    volatile int32_t lender[DS_MAX_SMS];
    volatile int32_t per_owner[2][DS_MAX_SMS];
    volatile int32_t per_lender[2][DS_MAX_SMS];
    volatile uint32_t ack_gen;        // device -> host: last host control generation installed
    volatile uint32_t fault_req[DS_MAX_TENANTS];  // host -> device: injected local exception code
    HostFault faults[DS_MAX_TENANTS];             // device -> host
};
constexpr int kHotGen = 0, kHotExit = 1, kHotPGen = 2, kHotFGen = 3, kHotTail = 64;
static_assert(kHotTail + DS_MAX_TENANTS <= 128, "tails fit the hot block");

struct DevState {
    DevTenant tenants[DS_MAX_TENANTS];
    DevControl ctl;
    // static configuration (written once by the host before ds_start)
    LaunchSlot* rings;             // device
    LaunchSlot* host_rings;        // host-mapped
    HostMailbox* mailbox;          // host-mapped
    HostCompletion* completions;   // host-mapped
    ds_block_record* blog;
    ds_switch_record* slog;
    ds_ctl_record* clog;
    uint32_t ring_mask;
    uint32_t completion_mask;
    unsigned long long blog_cap;
    unsigned long long slog_cap;
    unsigned long long clog_cap;
    uint32_t num_tenants_cap;
    uint32_t pad1;
    // device counters
    alignas(128) unsigned long long completion_count;
    alignas(128) unsigned long long blog_count;
    alignas(128) unsigned long long slog_count;
    alignas(128) unsigned long long clog_count;
    alignas(128) unsigned long long blocks_executed;
    // overhead ledger (OverheadLedger, engine.hpp:94-107) from device timestamps, per worker lane:
    //   switch: a lane's gap between its last block of one tenant and its first of another
    //   yield:  a lane finishing a block of a tenant its SM was revoked from, measured from
    //           the control install to that block's retire (the boundary wait)
    //   grant:  a lane's first block of a tenant after a control change, from the install
    alignas(128) unsigned long long led_switches;
    unsigned long long led_switch_ns, led_yields, led_yield_ns, led_grants, led_grant_ns;
    alignas(128) uint32_t trig_next;   // next armed trigger index
    uint32_t trig_count;
    ClaimTrigger* triggers;            // device array [kMaxTriggers]
    unsigned long long* retry;         // [DS_MAX_TENANTS][kRetryStride]
    float* save;                       // [abandonable tenants][kRetrySlots][kSaveFloats] spilled accumulators
    unsigned long long retry_mask;     // tenants that may abandon blocks (static)
    uint32_t drain_exit;               // loader exits once every enqueued launch completed (ds_set_drain_exit)
    uint32_t pad2;
    unsigned long long deadline_ns;    // loader exits this long after start (0: never)
    int32_t per_owner[2][DS_MAX_SMS];  // periodic program, cached from the mailbox
    int32_t per_lender[2][DS_MAX_SMS];
};

// Per-block context handed to a tenant body (the "unmodified kernel" sees
// only its logical block index and grid, never the physical SM).
struct BodyCtx {
    uint32_t bx, by, bz;
    uint32_t gx, gy, gz;
    const void* args;
    char* smem;          // dynamic shared memory (1024-aligned)
    uint32_t smem_bytes;
    uint32_t tmem_base;  // TMEM columns allocated for this CTA (0 if none)
    // Early-start dependency: launch `seq` of a tenant opens for claims as soon
    // as launch seq-1 is fully *claimed*; a block must not touch data produced
    // by earlier launches before wait_prev() (head >= seq).  Null in solo mode
    // (stream order already serialises launches).
    const uint32_t* prev_head;
    uint32_t seq;
    uint64_t* dbg;  // optional per-block phase timestamps (bodies that support it)
    // Local exceptions (raise_fault): the domain and tenant the block runs
    // for.  Null in solo mode.
    DevState* st;
    int32_t tenant;
    // Abandonable bodies set *abandon = 1 when they give the block up (the
    // scheduler then re-queues it instead of retiring it).  Null in solo mode.
    volatile uint32_t* abandon;
    // Spill/resume of abandoned tiles: *ab_info = (slot + 1) | (k << 16) of
    // the spill the body wrote (0: none); resume = the same for the spill
    // this block continues from (0: fresh start).
    volatile uint32_t* ab_info;
    uint32_t resume;
};

}  // namespace ds
