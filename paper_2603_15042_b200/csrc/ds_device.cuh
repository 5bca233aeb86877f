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

constexpr uint32_t kSat = 0x40000000u;      // claim-word block field >= kSat: kernel not open
constexpr int kBodyThreads = 256;           // warps 0..7 run tenant bodies
constexpr int kSchedWarp = 8;               // per-CTA scheduler warp (claims, retires, control)
constexpr int kLoaderWarp = 9;              // CTA 0 only: host mailbox poller
constexpr int kExecThreads = 320;
constexpr int kMaxArgs = 512;
constexpr uint32_t kDefaultSmem = 200 * 1024;
constexpr int kMaxTriggers = 64;

// Named barrier ids (0 is reserved for __syncthreads, 1 for body-internal syncs).
constexpr int kBarBody = 1;   // 256 body threads
constexpr int kBarFull = 2;   // scheduler staged work -> body
constexpr int kBarEmpty = 3;  // body copied the stage -> scheduler
constexpr int kBarDone = 4;   // body finished the block -> scheduler
constexpr int kBarExit = 5;
constexpr int kBarBody2 = 6;  // extra body-internal barrier ids for bodies (6..15)

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
    uint32_t pad[26];
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

struct alignas(128) DevControl {
    int32_t owner[DS_MAX_SMS];   // by physical smid
    int32_t lender[DS_MAX_SMS];
    uint32_t gen;                // bumped on every control change (any source)
    uint32_t exit;
    uint32_t pad[30];
};

struct HostCompletion {
    ds_completion c;
    volatile unsigned long long valid;  // index + 1 once c is written
    unsigned long long pad;
};
static_assert(sizeof(HostCompletion) == 64, "completion record is one line");

struct HostMailbox {
    volatile uint32_t gen;            // control generation written by host
    volatile uint32_t exit;
    volatile uint32_t periodic_gen;   // periodic program changed
    volatile uint32_t pad0;
    volatile unsigned long long periodic_ns;
    volatile uint32_t tail[DS_MAX_TENANTS];
    volatile int32_t owner[DS_MAX_SMS];   // by smid
    volatile int32_t lender[DS_MAX_SMS];
    volatile int32_t per_owner[2][DS_MAX_SMS];
    volatile int32_t per_lender[2][DS_MAX_SMS];
};

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
    alignas(128) uint32_t trig_next;   // next armed trigger index
    uint32_t trig_count;
    ClaimTrigger* triggers;            // device array [kMaxTriggers]
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
};

}  // namespace ds
