// Host side of the GPU-coroutine runtime: the C ABI of include/detshare/ds.h.
//
// One ds_domain = one GPU sharing domain (the reference's Device with its pctx
// pool, src/core/types.cpp:87-106).  The host owns registration (immutable
// kernel records, include/corosim/core/types.hpp:46-68), the pctx pool and the
// injective binding table (types.cpp:62-85), and writes the SM control word;
// the device executor (executor.cu) does everything per logical block.
//
// Threads: the caller's thread(s) issue API calls (serialised by a mutex); a
// drainer thread consumes device->host completion records from pinned mapped
// memory and maintains per-tenant completion state, transcripts and timings.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "ds_device.cuh"

extern "C" cudaError_t ds_dev_launch_executor(ds::DevState* st, int num_ctas, uint32_t smem, cudaStream_t s);
extern "C" cudaError_t ds_dev_executor_occupancy(uint32_t smem, int* blocks_per_sm);
extern "C" cudaError_t ds_dev_launch_solo(int body, const void* args, uint32_t gx, uint32_t gy, uint32_t gz,
                                          uint32_t smem, cudaStream_t s);
extern "C" cudaError_t ds_dev_probe(int nblocks, uint32_t* smids, uint32_t* nsmid, uint64_t* timer, cudaStream_t s);
extern "C" uint32_t ds_dev_body_smem(int body);
extern "C" int ds_dev_ctas_per_sm(void);

namespace {

thread_local std::string g_last_error;

int fail(int status, const std::string& why) {
    g_last_error = why;
    return status;
}

#define DS_CUDA(call)                                                                           \
    do {                                                                                        \
        cudaError_t _e = (call);                                                                \
        if (_e != cudaSuccess) return fail(DS_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

struct KernelRecord {
    std::string semantic_id;
    int body;
    uint32_t gx, gy, gz;
    uint32_t block_threads;
    uint64_t args_dev;   // device pointer into the arena
    std::vector<uint8_t> args_host;
    int phase;
    int64_t request;
    int decode_index;
    uint64_t fingerprint;
};

struct TenantRecord {
    std::string name;
    int priority;
    uint64_t next_seq = 0;            // launches issued
    uint64_t seen_at_stop = 0;        // launches the previous executor run had visible (ds_stop)
    std::atomic<uint64_t> completed{0};  // launches completed (drainer)
    std::vector<int32_t> launched_kernel;  // by seq
    std::vector<uint32_t> launched_grid;   // by seq (executed grid)
    int bound_pctx = -1;
};

struct Pctx {
    int64_t num, den;
    int n_sms;
    int bound = -1;              // tenant
    std::vector<int> slots;      // SM slots while bound
};

}  // namespace

struct ds_domain {
    int device = 0;
    int num_sms = 0;
    std::vector<int> smids;      // physical smid of slot i
    int nsmid = 0;
    uint32_t smem = ds::kDefaultSmem;
    int ring_cap = 1024;
    int lend_idle = 1;
    int lend_tenant = -1;
    int lane_split = 0;  // 1: owned SMs run the lend tenant on lane 1; 2: and lane 0 runs the owner only;
                         // 3, 4: as 1, 2 on every other owned SM

    cudaStream_t exec_stream = nullptr, copy_stream = nullptr;
    ds::DevState* d_state = nullptr;
    ds::LaunchSlot* d_rings = nullptr;
    ds::ClaimTrigger* d_triggers = nullptr;
    unsigned long long* d_retry = nullptr;   // [tenant][kRetryStride] abandoned blocks + occupancy hint
    unsigned long long retry_mask = 0;       // tenants whose blocks may be abandoned
    float* d_save = nullptr;                 // spilled accumulators of abandoned tiles
    int save_tenants = 0;
    uint8_t* d_args = nullptr;
    size_t args_cap = 0, args_used = 0;
    ds_block_record* d_blog = nullptr;
    ds_switch_record* d_slog = nullptr;
    ds_ctl_record* d_clog = nullptr;
    uint64_t blog_cap = 0, slog_cap = 1 << 20, clog_cap = 1 << 16;
    uint32_t* d_probe = nullptr;
    uint64_t* d_probe_t = nullptr;

    ds::HostMailbox* mb = nullptr;       // pinned mapped
    ds::LaunchSlot* h_rings = nullptr;   // pinned mapped
    ds::HostCompletion* h_comp = nullptr;
    uint32_t comp_cap = 1 << 18;

    std::vector<KernelRecord> kernels;
    std::vector<TenantRecord*> tenants;
    std::vector<Pctx> pctxs;
    std::vector<int32_t> owner, lender;  // by SM slot
    int n_triggers = 0;
    int prestart_triggers = 0;     // triggers installed while stopped: armed at the next ds_start
    int drain_exit = 0;            // executor exits once every enqueued launch completed
    uint64_t deadline_ms = 0;      // executor exits after this long (0: never)

    std::mutex mu;                 // API serialisation
    std::mutex comp_mu;            // completions vector
    std::condition_variable comp_cv;
    std::vector<ds_completion> completions;  // drained, not yet polled
    std::vector<std::vector<ds_completion>> per_tenant_done;
    std::atomic<bool> running{false};
    std::atomic<bool> drain_stop{false};
    std::thread drainer;
    uint64_t comp_next = 0;
    uint64_t enqueued = 0;
    std::atomic<uint64_t> completed_total{0};
};

namespace {

uint64_t fnv_mix(uint64_t h, uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);  // hash_mix, types.cpp:24-26
    return h;
}

// fingerprint over the immutable launch configuration (Kernel::fingerprint,
// types.cpp:39-48): semantic id, logical grid, body, argument block
uint64_t kernel_fingerprint(const KernelRecord& r, const uint8_t* args) {
    uint64_t h = 0x811c9dc5ULL;
    h = fnv_mix(h, r.semantic_id.size());
    for (unsigned char c : r.semantic_id) h = fnv_mix(h, c);
    h = fnv_mix(h, (uint64_t)r.gx * r.gy * r.gz);
    h = fnv_mix(h, (uint64_t)r.body);
    for (size_t i = 0; i < r.args_host.size(); ++i) h = fnv_mix(h, args[i]);
    return h;
}

// Host-side busy wait: the completion path is latency-critical (a decode
// step's completion gates the next step's launches), and a sleep costs the
// Linux timer slack (~50 us).  Poll with pause for a while after the last
// activity, then back off to short sleeps.
static inline void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#endif
}

void drain_loop(ds_domain* d) {
    auto last_active = std::chrono::steady_clock::now();
    while (!d->drain_stop.load(std::memory_order_acquire)) {
        bool any = false;
        for (;;) {
            ds::HostCompletion* hc = &d->h_comp[d->comp_next & (d->comp_cap - 1)];
            uint64_t v = hc->valid;
            if (v != d->comp_next + 1) break;
            std::atomic_thread_fence(std::memory_order_acquire);
            ds_completion c = hc->c;
            d->comp_next++;
            any = true;
            {
                std::lock_guard<std::mutex> g(d->comp_mu);
                d->completions.push_back(c);
                if (c.tenant >= 0 && c.tenant < (int)d->per_tenant_done.size())
                    d->per_tenant_done[c.tenant].push_back(c);
            }
            // monotonic: launch s+1's completion record can be written before
            // s's (s publishes head, then appends its record; a short s+1 may
            // retire in between), and s+1 done implies s done on the device
            if (c.tenant >= 0 && c.tenant < (int)d->tenants.size()) {
                auto& done = d->tenants[c.tenant]->completed;
                if (c.seq + 1 > done.load(std::memory_order_relaxed)) done.store(c.seq + 1, std::memory_order_release);
            }
            d->completed_total.fetch_add(1, std::memory_order_relaxed);
        }
        if (any) {
            d->comp_cv.notify_all();
            last_active = std::chrono::steady_clock::now();
        } else if (std::chrono::steady_clock::now() - last_active < std::chrono::milliseconds(20)) {
            for (int i = 0; i < 32; ++i) cpu_relax();
        } else {
            std::this_thread::sleep_for(std::chrono::microseconds(2));
        }
    }
}

// slot-space owner/lender -> smid-space control words (owner[], lender[] by smid)
void control_by_smid(ds_domain* d, volatile int32_t* owner_sm, volatile int32_t* lender_sm) {
    for (int i = 0; i < DS_MAX_SMS; ++i) {
        owner_sm[i] = -1;
        lender_sm[i] = -1;
    }
    for (int s = 0; s < d->num_sms; ++s) {
        int sm = d->smids[s];
        int32_t o = d->owner[s];
        int32_t l = d->lender[s];
        // idle-SM lending: only SMs bound to no pctx run the lend tenant; an
        // SM owned by a tenant never runs another tenant's blocks in its gaps
        // (a latency-critical owner would wait a whole foreign block on every
        // kernel boundary)
        if (d->lend_idle && l < 0 && o < 0 && d->lend_tenant >= 0) l = d->lend_tenant;
        // lane split: the owner's SMs also run the lend tenant on their second lane
        // (modes 3, 4: the same on every other owned SM only)
        if (d->lane_split && o >= 0 && d->lend_tenant >= 0 && d->lend_tenant != o &&
            (d->lane_split <= 2 || (s & 1))) {
            l = d->lend_tenant;
            o |= ds::kCtlSplit | (d->lane_split % 2 == 0 ? ds::kCtlOwnerOnly0 : 0);
        }
        owner_sm[sm] = o;
        lender_sm[sm] = l;
    }
}

int push_control(ds_domain* d) {
    // slot-space owner/lender -> smid-space mailbox (full arrays and the
    // compact tagged image the loader installs from its poll), then bump the
    // generation
    control_by_smid(d, d->mb->owner, d->mb->lender);
    const uint32_t gen = d->mb->hot[ds::kHotGen] + 1;
    const uint32_t tag = (gen & 0xffffu) << 16;
    for (int i = 0; i < DS_MAX_SMS; ++i) {
        const int32_t o = d->mb->owner[i], l = d->mb->lender[i];
        const uint32_t ot = o < 0 ? ds::kImgNone : (uint32_t)(o & ds::kCtlTenantMask) & 0x3fu;
        const uint32_t lt = l < 0 ? ds::kImgNone : (uint32_t)l & 0x3fu;
        const uint32_t fl = o < 0 ? 0u : (((o & ds::kCtlSplit) ? 1u : 0u) << 14) | (((o & ds::kCtlOwnerOnly0) ? 1u : 0u) << 15);
        d->mb->ctl_img[i] = tag | fl | (lt << 7) | ot;
    }
    std::atomic_thread_fence(std::memory_order_seq_cst);
    d->mb->hot[ds::kHotGen] = gen;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    return DS_OK;
}

// Choose n free SM slots, preferring whole TPCs (slot pairs with smid 2k,2k+1).
std::vector<int> pick_slots(ds_domain* d, int n) {
    std::vector<int> free_slots;
    for (int s = 0; s < d->num_sms; ++s)
        if (d->owner[s] < 0) free_slots.push_back(s);
    std::sort(free_slots.begin(), free_slots.end(), [&](int a, int b) { return d->smids[a] < d->smids[b]; });
    std::vector<int> out;
    for (int s : free_slots) {
        if ((int)out.size() >= n) break;
        out.push_back(s);
    }
    return out;
}

// The device keeps 32-bit launch sequence numbers; widen one against the
// host's 64-bit count (it is at most 2^32 behind).
uint64_t widen_seq(uint64_t host_next, uint32_t dev) {
    uint64_t v = (host_next & ~0xffffffffull) | dev;
    if (v > host_next) v -= 1ull << 32;
    return v;
}

// Launch seq of a tenant will never complete intact (local exception).
bool seq_failed(ds_domain* d, int tenant, uint64_t seq) {
    const ds::HostFault& f = d->mb->faults[tenant];
    if (!f.code) return false;
    std::atomic_thread_fence(std::memory_order_acquire);
    return seq >= widen_seq(d->tenants[tenant]->next_seq, f.head);
}

int check_dom(ds_domain* d) {
    if (!d) return fail(DS_INVALID_ARGUMENT, "null domain");
    return DS_OK;
}

}  // namespace

extern "C" {

const char* ds_status_name(int status) {
    switch (status) {
        case DS_OK: return "Ok";
        case DS_INVALID_TIER: return "InvalidTier";
        case DS_BIND_CONFLICT: return "BindConflict";
        case DS_DOUBLE_BIND: return "DoubleBind";
        case DS_CAUSALITY_VIOLATION: return "CausalityViolation";
        case DS_EVENT_BUDGET_EXCEEDED: return "EventBudgetExceeded";
        case DS_TRACE_VIOLATION: return "TraceViolation";
        case DS_PLAN_MISMATCH: return "PlanMismatch";
        case DS_INVALID_SPLIT: return "InvalidSplit";
        case DS_PARSE_ERROR: return "ParseError";
        case DS_CONFIG_ERROR: return "ConfigError";
        case DS_CUDA_ERROR: return "CudaError";
        case DS_NO_DEVICE: return "NoDevice";
        case DS_NOT_RUNNING: return "NotRunning";
        case DS_TIMEOUT: return "Timeout";
        case DS_RING_FULL: return "RingFull";
        case DS_INVALID_ARGUMENT: return "InvalidArgument";
        case DS_ALREADY_RUNNING: return "AlreadyRunning";
        case DS_TENANT_FAILED: return "TenantFailed";
        case DS_RECORD_MUTATED: return "RecordMutated";
    }
    return "UnknownError";  // errors.cpp:19
}

const char* ds_last_error(void) { return g_last_error.c_str(); }
int ds_abi_version(void) { return DS_ABI_VERSION; }

int ds_body_smem(int body, uint32_t* bytes) {
    if (!bytes || body <= 0 || body >= DS_BODY_COUNT) return fail(DS_INVALID_ARGUMENT, "unknown body");
    *bytes = ds_dev_body_smem(body);
    return DS_OK;
}

int ds_domain_create(const ds_domain_config* cfg, ds_domain** out) {
    if (!cfg || !out) return fail(DS_INVALID_ARGUMENT, "null config");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(DS_NO_DEVICE, "no CUDA device");
    if (cfg->device < 0 || cfg->device >= ndev) return fail(DS_NO_DEVICE, "bad device ordinal");
    if (cfg->n_tiers < 1 || cfg->n_tiers > 16) return fail(DS_INVALID_TIER, "pool needs 1..16 tiers");
    for (int i = 0; i < cfg->n_tiers; ++i) {
        // create_pool (types.cpp:87-98): tiers must lie in (0, 1]
        if (cfg->tier_den[i] <= 0 || cfg->tier_num[i] <= 0 || cfg->tier_num[i] > cfg->tier_den[i])
            return fail(DS_INVALID_TIER, "tier fraction outside (0, 1]");
    }
    int ring = cfg->ring_capacity > 0 ? cfg->ring_capacity : 1024;
    if ((ring & (ring - 1)) != 0 || ring > 4096) return fail(DS_CONFIG_ERROR, "ring_capacity must be a power of two <= 4096");

    auto* d = new ds_domain();
    d->device = cfg->device;
    d->ring_cap = ring;
    d->lend_idle = cfg->lend_idle_sms;
    if (cfg->executor_smem > 0) d->smem = (uint32_t)cfg->executor_smem;
    d->blog_cap = cfg->block_log_capacity > 0 ? (uint64_t)cfg->block_log_capacity : 0;
    auto bail = [&](int st) {
        delete d;
        return st;
    };
    if (cudaSetDevice(d->device) != cudaSuccess) return bail(fail(DS_CUDA_ERROR, "cudaSetDevice"));
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, d->device);
    if (prop.major < 10) return bail(fail(DS_NO_DEVICE, "needs sm_100 (B200)"));
    d->num_sms = prop.multiProcessorCount;
    if (d->num_sms > DS_MAX_SMS) return bail(fail(DS_CONFIG_ERROR, "too many SMs"));
    int occ = 0;
    if (ds_dev_executor_occupancy(d->smem, &occ) != cudaSuccess || occ != ds_dev_ctas_per_sm())
        return bail(fail(DS_CONFIG_ERROR, "executor must be exactly " + std::to_string(ds_dev_ctas_per_sm()) +
                                              " CTA(s)/SM (occupancy " + std::to_string(occ) + ")"));

    cudaStreamCreateWithFlags(&d->exec_stream, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&d->copy_stream, cudaStreamNonBlocking);

    // probe %smid of each SM (many CTAs, take the distinct set)
    {
        int nb = d->num_sms * 8;
        uint32_t *dsm = nullptr, *dn = nullptr;
        uint64_t* dt = nullptr;
        cudaMalloc(&dsm, nb * sizeof(uint32_t));
        cudaMalloc(&dn, sizeof(uint32_t));
        cudaMalloc(&dt, sizeof(uint64_t));
        ds_dev_probe(nb, dsm, dn, dt, d->copy_stream);
        std::vector<uint32_t> h(nb);
        uint32_t nsmid = 0;
        cudaMemcpyAsync(h.data(), dsm, nb * sizeof(uint32_t), cudaMemcpyDeviceToHost, d->copy_stream);
        cudaMemcpyAsync(&nsmid, dn, sizeof(uint32_t), cudaMemcpyDeviceToHost, d->copy_stream);
        cudaError_t e = cudaStreamSynchronize(d->copy_stream);
        cudaFree(dsm);
        cudaFree(dn);
        cudaFree(dt);
        if (e != cudaSuccess) return bail(fail(DS_CUDA_ERROR, std::string("probe: ") + cudaGetErrorString(e)));
        std::sort(h.begin(), h.end());
        h.erase(std::unique(h.begin(), h.end()), h.end());
        d->nsmid = (int)nsmid;
        if ((int)h.size() != d->num_sms || nsmid > DS_MAX_SMS)
            return bail(fail(DS_CONFIG_ERROR, "smid probe saw " + std::to_string(h.size()) + " SMs, nsmid " +
                                                  std::to_string(nsmid)));
        for (uint32_t s : h) d->smids.push_back((int)s);
    }
    d->owner.assign(d->num_sms, -1);
    d->lender.assign(d->num_sms, -1);

    // pool (create_pool): one pctx per tier; SM count = floor(tier * num_sms),
    // >= 1, so every set of pctxs the policy may bind together (sum of tiers
    // <= 1, engine.cpp:721-725) also fits in the SMs (rounding up could not)
    for (int i = 0; i < cfg->n_tiers; ++i) {
        Pctx p;
        p.num = cfg->tier_num[i];
        p.den = cfg->tier_den[i];
        p.n_sms = (int)(p.num * d->num_sms / p.den);
        if (p.n_sms < 1) p.n_sms = 1;
        if (p.n_sms > d->num_sms) p.n_sms = d->num_sms;
        d->pctxs.push_back(p);
    }

    // device memory
    size_t ring_bytes = sizeof(ds::LaunchSlot) * DS_MAX_TENANTS * (size_t)ring;
    d->args_cap = 8u << 20;
    if (cudaMalloc(&d->d_state, sizeof(ds::DevState)) != cudaSuccess ||
        cudaMalloc(&d->d_rings, ring_bytes) != cudaSuccess || cudaMalloc(&d->d_args, d->args_cap) != cudaSuccess ||
        cudaMalloc(&d->d_triggers, sizeof(ds::ClaimTrigger) * ds::kMaxTriggers) != cudaSuccess ||
        cudaMalloc(&d->d_retry, sizeof(unsigned long long) * DS_MAX_TENANTS * ds::kRetryStride) != cudaSuccess ||
        cudaMalloc(&d->d_slog, sizeof(ds_switch_record) * d->slog_cap) != cudaSuccess ||
        cudaMalloc(&d->d_clog, sizeof(ds_ctl_record) * d->clog_cap) != cudaSuccess)
        return bail(fail(DS_CUDA_ERROR, "cudaMalloc"));
    if (cudaMalloc(&d->d_probe, 16) != cudaSuccess || cudaMalloc(&d->d_probe_t, 8) != cudaSuccess)
        return bail(fail(DS_CUDA_ERROR, "cudaMalloc probe"));
    if (d->blog_cap && cudaMalloc(&d->d_blog, sizeof(ds_block_record) * d->blog_cap) != cudaSuccess)
        return bail(fail(DS_CUDA_ERROR, "cudaMalloc block log"));
    // host mapped
    if (cudaHostAlloc(&d->mb, sizeof(ds::HostMailbox), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
        cudaHostAlloc(&d->h_rings, ring_bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
        cudaHostAlloc(&d->h_comp, sizeof(ds::HostCompletion) * d->comp_cap,
                      cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
        return bail(fail(DS_CUDA_ERROR, "cudaHostAlloc"));
    std::memset((void*)d->mb, 0, sizeof(ds::HostMailbox));
    std::memset(d->h_rings, 0, ring_bytes);
    std::memset(d->h_comp, 0, sizeof(ds::HostCompletion) * d->comp_cap);
    for (int i = 0; i < DS_MAX_SMS; ++i) {
        d->mb->owner[i] = -1;
        d->mb->lender[i] = -1;
    }
    *out = d;
    return DS_OK;
}

int ds_domain_destroy(ds_domain* d) {
    if (!d) return DS_OK;
    if (d->running) ds_stop(d);
    cudaSetDevice(d->device);
    cudaFree(d->d_state);
    cudaFree(d->d_rings);
    cudaFree(d->d_args);
    cudaFree(d->d_triggers);
    cudaFree(d->d_retry);
    cudaFree(d->d_save);
    cudaFree(d->d_slog);
    cudaFree(d->d_clog);
    if (d->d_blog) cudaFree(d->d_blog);
    cudaFree(d->d_probe);
    cudaFree(d->d_probe_t);
    cudaFreeHost((void*)d->mb);
    cudaFreeHost(d->h_rings);
    cudaFreeHost(d->h_comp);
    if (d->exec_stream) cudaStreamDestroy(d->exec_stream);
    if (d->copy_stream) cudaStreamDestroy(d->copy_stream);
    for (auto* t : d->tenants) delete t;
    delete d;
    return DS_OK;
}

int ds_num_sms(ds_domain* d, int* out) {
    if (check_dom(d) || !out) return fail(DS_INVALID_ARGUMENT, "null");
    *out = d->num_sms;
    return DS_OK;
}

int ds_smids(ds_domain* d, int* out, int cap, int* n) {
    if (check_dom(d) || !n) return fail(DS_INVALID_ARGUMENT, "null");
    int m = std::min(cap, d->num_sms);
    for (int i = 0; i < m; ++i) out[i] = d->smids[i];
    *n = d->num_sms;
    return DS_OK;
}

int ds_pctx_count(ds_domain* d, int* out) {
    if (check_dom(d) || !out) return fail(DS_INVALID_ARGUMENT, "null");
    *out = (int)d->pctxs.size();
    return DS_OK;
}

int ds_pctx_info(ds_domain* d, int pctx, int64_t* num, int64_t* den, int* n_sms, int* bound) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> g(d->mu);
    if (pctx < 0 || pctx >= (int)d->pctxs.size()) return fail(DS_INVALID_ARGUMENT, "unknown pctx");
    const Pctx& p = d->pctxs[pctx];
    if (num) *num = p.num;
    if (den) *den = p.den;
    if (n_sms) *n_sms = p.n_sms;
    if (bound) *bound = p.bound;
    return DS_OK;
}

int ds_tenant_register(ds_domain* d, const ds_tenant_desc* desc, int* tenant_id) {
    if (check_dom(d) || !desc || !tenant_id) return fail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(d->mu);
    if ((int)d->tenants.size() >= DS_MAX_TENANTS) return fail(DS_CONFIG_ERROR, "too many tenants");
    auto* t = new TenantRecord();
    t->name = desc->name ? desc->name : "";
    t->priority = desc->priority;
    d->tenants.push_back(t);
    {
        std::lock_guard<std::mutex> g2(d->comp_mu);
        d->per_tenant_done.emplace_back();
    }
    *tenant_id = (int)d->tenants.size() - 1;  // job i => vctx i (engine.cpp:139-145)
    return DS_OK;
}

int ds_kernel_register(ds_domain* d, const ds_kernel_desc* k, int* kernel_id) {
    if (check_dom(d) || !k || !kernel_id) return fail(DS_INVALID_ARGUMENT, "null");
    if (k->body <= DS_BODY_NONE || k->body >= DS_BODY_COUNT) return fail(DS_CONFIG_ERROR, "unknown body");
    uint64_t grid = (uint64_t)k->grid_x * k->grid_y * k->grid_z;
    if (grid < 1 || grid >= ds::kSat) return fail(DS_CONFIG_ERROR, "grid_size must be >= 1");  // engine.cpp:169-171
    if (k->block_threads != 256) return fail(DS_CONFIG_ERROR, "built-in bodies run 256 threads");
    if (k->args_size > ds::kMaxArgs || (k->args_size && !k->args)) return fail(DS_CONFIG_ERROR, "args too large");
    if (k->body == DS_BODY_GEMM_BF16 && k->args_size >= ds::kGemmArgsBody) {
        // abandonable tiles are queued as ((seq+1) << 32) | (k << 20) | block:
        // the logical block must fit 20 bits and the resume k-block 12 bits
        int32_t K = 0, bk = 0, ab = 0;
        std::memcpy(&K, (const uint8_t*)k->args + ds::kGemmArgsOffK, 4);
        std::memcpy(&bk, (const uint8_t*)k->args + ds::kGemmArgsOffBk, 4);
        std::memcpy(&ab, (const uint8_t*)k->args + ds::kGemmArgsOffAbandon, 4);
        if (ab && (grid >= (1ull << ds::kRetryBlockBits) || K / (bk > 0 ? bk : 64) >= 4096))
            return fail(DS_CONFIG_ERROR, "abandonable GEMM needs grid < 2^20 and K/bk < 4096");
    }
    std::lock_guard<std::mutex> g(d->mu);
    if (d->args_used + ds::kMaxArgs > d->args_cap) return fail(DS_CONFIG_ERROR, "args arena full");
    KernelRecord r;
    r.semantic_id = k->semantic_id ? k->semantic_id : "";
    r.body = k->body;
    r.gx = k->grid_x;
    r.gy = k->grid_y;
    r.gz = k->grid_z;
    r.block_threads = k->block_threads;
    r.args_dev = (uint64_t)(d->d_args + d->args_used);
    r.args_host.assign((const uint8_t*)k->args, (const uint8_t*)k->args + k->args_size);
    r.phase = k->phase;
    r.request = k->request;
    r.decode_index = k->decode_index;
    r.fingerprint = kernel_fingerprint(r, r.args_host.data());
    if (k->args_size) {
        cudaSetDevice(d->device);
        DS_CUDA(cudaMemcpyAsync((void*)r.args_dev, k->args, k->args_size, cudaMemcpyHostToDevice, d->copy_stream));
        DS_CUDA(cudaStreamSynchronize(d->copy_stream));
    }
    d->args_used += ds::kMaxArgs;
    d->kernels.push_back(std::move(r));
    *kernel_id = (int)d->kernels.size() - 1;
    return DS_OK;
}

int ds_start(ds_domain* d) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> g(d->mu);
    if (d->running) return fail(DS_ALREADY_RUNNING, "executor already running");
    cudaSetDevice(d->device);
    ds::DevState h;
    std::memset(&h, 0, sizeof(h));
    for (int t = 0; t < DS_MAX_TENANTS; ++t) {
        uint64_t seq = t < (int)d->tenants.size() ? d->tenants[t]->next_seq : 0;
        uint64_t done = t < (int)d->tenants.size() ? d->tenants[t]->completed.load() : 0;
        const uint32_t fault = d->mb->faults[t].code;
        if (fault) {  // a failed tenant stays failed across restarts
            h.tenants[t].fault = fault;
            h.tenants[t].claim = ((unsigned long long)seq << 32) | ds::kDead;
            h.tenants[t].tail = (uint32_t)seq;
            h.tenants[t].head = (uint32_t)done;
            d->mb->hot[ds::kHotTail + t] = (uint32_t)seq;
            continue;
        }
        // launches a previous run saw must all have completed (a half-run
        // launch cannot resume across executor restarts); launches enqueued
        // while stopped (seq >= seen_at_stop) are picked up by the loader
        const uint64_t seen = t < (int)d->tenants.size() ? d->tenants[t]->seen_at_stop : 0;
        if (done != seen) return fail(DS_CONFIG_ERROR, "tenant has launches in flight from a previous run");
        h.tenants[t].claim = ((unsigned long long)done << 32) | ds::kSat;
        h.tenants[t].tail = (uint32_t)done;
        h.tenants[t].head = (uint32_t)done;
        d->mb->hot[ds::kHotTail + t] = (uint32_t)seq;
    }
    // the control word in force at launch (installed before the kernel runs,
    // so a pre-enqueued program needs no host round trip)
    {
        int32_t o[DS_MAX_SMS], l[DS_MAX_SMS];
        control_by_smid(d, o, l);
        for (int i = 0; i < DS_MAX_SMS; ++i)
            h.ctl.word[i] = ((unsigned long long)(uint32_t)l[i] << 32) | (uint32_t)o[i];
    }
    h.drain_exit = (uint32_t)d->drain_exit;
    h.deadline_ns = d->deadline_ms * 1000000ull;
    h.rings = d->d_rings;
    ds::LaunchSlot* hr = nullptr;
    ds::HostMailbox* hm = nullptr;
    ds::HostCompletion* hc = nullptr;
    DS_CUDA(cudaHostGetDevicePointer((void**)&hr, d->h_rings, 0));
    DS_CUDA(cudaHostGetDevicePointer((void**)&hm, (void*)d->mb, 0));
    DS_CUDA(cudaHostGetDevicePointer((void**)&hc, d->h_comp, 0));
    h.host_rings = hr;
    h.mailbox = hm;
    h.completions = hc;
    h.blog = d->d_blog;
    h.slog = d->d_slog;
    h.clog = d->d_clog;
    h.ring_mask = (uint32_t)d->ring_cap - 1;
    h.completion_mask = d->comp_cap - 1;
    h.blog_cap = d->blog_cap;
    h.slog_cap = d->slog_cap;
    h.clog_cap = d->clog_cap;
    h.num_tenants_cap = DS_MAX_TENANTS;
    h.triggers = d->d_triggers;
    h.retry = d->d_retry;
    h.retry_mask = d->retry_mask;
    // a tenant's retry ring holds at most one abandoned block per worker lane
    if (d->retry_mask && d->num_sms * ds::kLanes > ds::kRetrySlots)
        return fail(DS_CONFIG_ERROR, "abandonable tenants need num_sms x lanes <= retry-ring slots");
    {
        const int n_ab = __builtin_popcountll(d->retry_mask);
        if (n_ab != d->save_tenants) {
            cudaFree(d->d_save);
            d->d_save = nullptr;
            d->save_tenants = 0;
            if (n_ab) {
                DS_CUDA(cudaMalloc(&d->d_save, sizeof(float) * (size_t)n_ab * ds::kRetrySlots * ds::kSaveFloats));
                d->save_tenants = n_ab;
            }
        }
        int rank = 0;
        for (int t = 0; t < DS_MAX_TENANTS; ++t)
            if ((d->retry_mask >> t) & 1ull) h.tenants[t].save_base = (uint32_t)(rank++ * ds::kRetrySlots);
        h.save = d->d_save;
    }
    DS_CUDA(cudaMemsetAsync(d->d_retry, 0, sizeof(unsigned long long) * DS_MAX_TENANTS * ds::kRetryStride,
                            d->copy_stream));
    // triggers installed while stopped are armed for this run; others reset
    h.trig_count = (uint32_t)d->prestart_triggers;
    h.trig_next = 0;
    d->n_triggers = d->prestart_triggers;
    d->prestart_triggers = 0;
    // completions restart from index 0
    std::memset(d->h_comp, 0, sizeof(ds::HostCompletion) * d->comp_cap);
    d->comp_next = 0;
    d->mb->hot[ds::kHotExit] = 0;
    d->mb->periodic_ns = 0;
    d->mb->hot[ds::kHotGen] = 0;
    d->mb->hot[ds::kHotFGen] = 0;
    DS_CUDA(cudaMemcpyAsync(d->d_state, &h, sizeof(h), cudaMemcpyHostToDevice, d->copy_stream));
    DS_CUDA(cudaStreamSynchronize(d->copy_stream));
    d->drain_stop = false;
    d->drainer = std::thread(drain_loop, d);
    cudaError_t e = ds_dev_launch_executor(d->d_state, d->num_sms * ds_dev_ctas_per_sm(), d->smem, d->exec_stream);
    if (e != cudaSuccess) {
        d->drain_stop = true;
        d->drainer.join();
        return fail(DS_CUDA_ERROR, std::string("executor launch: ") + cudaGetErrorString(e));
    }
    d->running = true;
    push_control(d);
    return DS_OK;
}

int ds_set_drain_exit(ds_domain* d, int enable, uint64_t deadline_ms) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> g(d->mu);
    if (d->running) return fail(DS_ALREADY_RUNNING, "set before ds_start");
    d->drain_exit = enable ? 1 : 0;
    d->deadline_ms = deadline_ms;
    return DS_OK;
}

int ds_stop(ds_domain* d) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> g(d->mu);
    if (!d->running) return DS_OK;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    d->mb->hot[ds::kHotExit] = 1;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    cudaSetDevice(d->device);
    // bounded wait: a wedged tenant body must not hang the caller forever
    cudaError_t e = cudaErrorNotReady;
    auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(20);
    while ((e = cudaStreamQuery(d->exec_stream)) == cudaErrorNotReady) {
        if (std::chrono::steady_clock::now() > deadline) {
            d->drain_stop = true;
            d->drainer.join();
            return fail(DS_TIMEOUT, "executor did not exit within 20 s");
        }
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    // drain what is left, then stop the drainer
    std::this_thread::sleep_for(std::chrono::milliseconds(1));
    d->drain_stop = true;
    d->drainer.join();
    d->running = false;
    for (auto* t : d->tenants) t->seen_at_stop = t->next_seq;
    if (e != cudaSuccess) return fail(DS_CUDA_ERROR, std::string("executor: ") + cudaGetErrorString(e));
    return DS_OK;
}

static int launch_impl(ds_domain* d, int tenant, int kernel_id, uint64_t tag, uint32_t exec_grid, uint32_t egx,
                       uint32_t egy, uint32_t egz, uint64_t* seq_out, uint32_t start = 0) {
    if (start >= exec_grid) return fail(DS_INVALID_ARGUMENT, "resume block beyond the grid");
    if (tenant < 0 || tenant >= (int)d->tenants.size()) return fail(DS_INVALID_ARGUMENT, "unknown tenant");
    if (kernel_id < 0 || kernel_id >= (int)d->kernels.size()) return fail(DS_INVALID_ARGUMENT, "unknown kernel");
    TenantRecord* t = d->tenants[tenant];
    const KernelRecord& k = d->kernels[kernel_id];
    uint64_t seq = t->next_seq;
    // arrivals of a failed vctx are dropped (engine.cpp:810-819)
    if (d->mb->faults[tenant].code) return fail(DS_TENANT_FAILED, "tenant failed (local exception)");
    // ring flow control: slot seq % R is free once seq - R completed
    auto t0 = std::chrono::steady_clock::now();
    while (seq - t->completed.load(std::memory_order_acquire) >= (uint64_t)d->ring_cap) {
        if (!d->running) return fail(DS_RING_FULL, "ring full and executor stopped");
        if (d->mb->faults[tenant].code) return fail(DS_TENANT_FAILED, "tenant failed (local exception)");
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30)) return fail(DS_RING_FULL, "ring full");
        std::this_thread::yield();
    }
    ds::LaunchSlot& s = d->h_rings[(size_t)tenant * d->ring_cap + (seq & (d->ring_cap - 1))];
    s.body = k.body;
    s.grid = exec_grid;
    s.gx = egx;
    s.gy = egy;
    s.gz = egz;
    s.kernel_id = kernel_id;
    s.args = k.args_dev;
    s.tag = tag;
    s.retired = start;  // blocks below `start` ran before a migration: they count as retired
    s.sms = 0;
    s.t_first = 0;
    s.seq = (uint32_t)seq;
    s.flags = start;    // first logical block the executor hands out
    t->launched_kernel.push_back(kernel_id);
    t->launched_grid.push_back(exec_grid);
    t->next_seq = seq + 1;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    d->mb->hot[ds::kHotTail + tenant] = (uint32_t)(seq + 1);
    std::atomic_thread_fence(std::memory_order_seq_cst);
    d->enqueued++;
    if (seq_out) *seq_out = seq;
    return DS_OK;
}

int ds_launch(ds_domain* d, int tenant, int kernel_id, uint64_t tag, uint64_t* seq) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> g(d->mu);
    if (kernel_id < 0 || kernel_id >= (int)d->kernels.size()) return fail(DS_INVALID_ARGUMENT, "unknown kernel");
    const KernelRecord& k = d->kernels[kernel_id];
    return launch_impl(d, tenant, kernel_id, tag, k.gx * k.gy * k.gz, k.gx, k.gy, k.gz, seq);
}

int ds_launch_from(ds_domain* d, int tenant, int kernel_id, uint64_t tag, uint32_t first_block, uint64_t* seq) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> g(d->mu);
    if (kernel_id < 0 || kernel_id >= (int)d->kernels.size()) return fail(DS_INVALID_ARGUMENT, "unknown kernel");
    const KernelRecord& k = d->kernels[kernel_id];
    return launch_impl(d, tenant, kernel_id, tag, k.gx * k.gy * k.gz, k.gx, k.gy, k.gz, seq, first_block);
}

int ds_tenant_progress(ds_domain* d, int tenant, ds_progress* out) {
    if (check_dom(d) || !out) return fail(DS_INVALID_ARGUMENT, "null");
    if (tenant < 0 || tenant >= (int)d->tenants.size()) return fail(DS_INVALID_ARGUMENT, "unknown tenant");
    cudaSetDevice(d->device);
    ds::DevTenant T;
    DS_CUDA(cudaMemcpyAsync(&T, &d->d_state->tenants[tenant], sizeof T, cudaMemcpyDeviceToHost, d->copy_stream));
    DS_CUDA(cudaStreamSynchronize(d->copy_stream));
    std::memset(out, 0, sizeof *out);
    out->head = T.head;
    out->tail = T.tail;
    out->enqueued = d->tenants[tenant]->next_seq;
    out->claim_seq = (uint32_t)(T.claim >> 32);
    const uint32_t b = (uint32_t)T.claim;
    out->claim_open = b < ds::kSat;
    out->failed = (b & ds::kDead) != 0 || T.fault != 0;
    if (out->claim_open && out->claim_seq < T.tail) {
        ds::LaunchSlot sl;
        const size_t idx = (size_t)tenant * d->ring_cap + (out->claim_seq & (d->ring_cap - 1));
        DS_CUDA(cudaMemcpyAsync(&sl, d->d_rings + idx, sizeof sl, cudaMemcpyDeviceToHost, d->copy_stream));
        DS_CUDA(cudaStreamSynchronize(d->copy_stream));
        out->claim_block = std::min(b, sl.grid);
        out->claim_grid = sl.grid;
        out->claim_retired = sl.retired;
    }
    // quiescent: every launch before the claimed one completed and every
    // claimed block of it retired (no block of the tenant is running)
    out->drained = T.head == out->claim_seq && (!out->claim_open || out->claim_retired == out->claim_block);
    return DS_OK;
}

// atomized_grid (engine.cpp:26-30): the grid is rewritten to fit the tier.
int ds_launch_atomized(ds_domain* d, int tenant, int kernel_id, uint64_t tag, int64_t num, int64_t den,
                       uint64_t* seq) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    if (den <= 0 || num <= 0 || num > den) return fail(DS_INVALID_TIER, "tier outside (0, 1]");
    std::lock_guard<std::mutex> g(d->mu);
    if (kernel_id < 0 || kernel_id >= (int)d->kernels.size()) return fail(DS_INVALID_ARGUMENT, "unknown kernel");
    const KernelRecord& k = d->kernels[kernel_id];
    uint64_t grid = (uint64_t)k.gx * k.gy * k.gz;
    int64_t gnew = (int64_t)(grid * (uint64_t)num / (uint64_t)den);
    if (gnew < 1) gnew = 1;
    // 1-D rewrite of the logical grid (the mutant breaks the launch config by design)
    return launch_impl(d, tenant, kernel_id, tag, (uint32_t)gnew, (uint32_t)gnew, 1, 1, seq);
}

int ds_wait_tenant(ds_domain* d, int tenant, uint64_t seq, int timeout_ms) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    if (tenant < 0 || tenant >= (int)d->tenants.size()) return fail(DS_INVALID_ARGUMENT, "unknown tenant");
    TenantRecord* t = d->tenants[tenant];
    auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms < 0 ? 1 << 30 : timeout_ms);
    for (;;) {
        if (seq_failed(d, tenant, seq)) return fail(DS_TENANT_FAILED, "tenant failed (local exception)");
        if (t->completed.load(std::memory_order_acquire) > seq) break;
        if (!d->running) return fail(DS_NOT_RUNNING, "executor not running");
        if (std::chrono::steady_clock::now() > deadline) return fail(DS_TIMEOUT, "wait timed out");
        std::unique_lock<std::mutex> lk(d->comp_mu);
        d->comp_cv.wait_for(lk, std::chrono::microseconds(200));
    }
    return DS_OK;
}

int ds_fault_inject(ds_domain* d, int tenant, uint32_t code) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    if (tenant < 0 || tenant >= (int)d->tenants.size()) return fail(DS_INVALID_ARGUMENT, "unknown tenant");
    if (code == 0) return fail(DS_INVALID_ARGUMENT, "fault code must be nonzero");
    std::lock_guard<std::mutex> g(d->mu);
    if (d->mb->faults[tenant].code) return DS_OK;  // first fault wins
    if (!d->running) {  // nothing on the device: record it directly
        ds::HostFault& f = d->mb->faults[tenant];
        f.seq = (uint32_t)d->tenants[tenant]->next_seq;
        f.head = (uint32_t)d->tenants[tenant]->completed.load();
        f.block = 0xffffffffu;
        f.t = 0;
        std::atomic_thread_fence(std::memory_order_seq_cst);
        f.code = code;
        return DS_OK;
    }
    d->mb->fault_req[tenant] = code;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    d->mb->hot[ds::kHotFGen] = d->mb->hot[ds::kHotFGen] + 1;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    // the loader applies it within one poll; return once it is visible
    auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(5);
    while (!d->mb->faults[tenant].code) {
        if (std::chrono::steady_clock::now() > deadline) return fail(DS_TIMEOUT, "fault not acknowledged");
        std::this_thread::yield();
    }
    return DS_OK;
}

int ds_tenant_fault(ds_domain* d, int tenant, ds_fault_info* out) {
    if (check_dom(d) || !out) return fail(DS_INVALID_ARGUMENT, "null");
    if (tenant < 0 || tenant >= (int)d->tenants.size()) return fail(DS_INVALID_ARGUMENT, "unknown tenant");
    const ds::HostFault& f = d->mb->faults[tenant];
    std::memset(out, 0, sizeof(*out));
    const uint32_t c = f.code;
    std::atomic_thread_fence(std::memory_order_acquire);
    if (!c) return DS_OK;
    out->code = c;
    out->block = f.block;
    out->seq = widen_seq(d->tenants[tenant]->next_seq, f.seq);
    out->first_failed = widen_seq(d->tenants[tenant]->next_seq, f.head);
    out->t_ns = f.t;
    return DS_OK;
}

int ds_poll(ds_domain* d, ds_completion* out, int cap, int* n) {
    if (check_dom(d) || !n) return fail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(d->comp_mu);
    int m = std::min<int>(cap, (int)d->completions.size());
    for (int i = 0; i < m; ++i) out[i] = d->completions[i];
    d->completions.erase(d->completions.begin(), d->completions.begin() + m);
    *n = m;
    return DS_OK;
}

int ds_quota_set(ds_domain* d, const int32_t* owner, const int32_t* lender, int n) {
    if (check_dom(d) || n != d->num_sms) return fail(DS_INVALID_ARGUMENT, "control word needs num_sms entries");
    std::lock_guard<std::mutex> g(d->mu);
    for (int i = 0; i < n; ++i) {
        d->owner[i] = owner ? owner[i] : -1;
        d->lender[i] = lender ? lender[i] : -1;
    }
    // raw control bypasses the pctx table: forget bindings
    for (auto& p : d->pctxs) {
        if (p.bound >= 0) d->tenants[p.bound]->bound_pctx = -1;
        p.bound = -1;
        p.slots.clear();
    }
    return push_control(d);
}

int ds_quota_get(ds_domain* d, int32_t* owner, int32_t* lender, int n) {
    if (check_dom(d) || n != d->num_sms) return fail(DS_INVALID_ARGUMENT, "control word needs num_sms entries");
    std::lock_guard<std::mutex> g(d->mu);
    for (int i = 0; i < n; ++i) {
        if (owner) owner[i] = d->owner[i];
        if (lender) lender[i] = d->lender[i];
    }
    return DS_OK;
}

int ds_set_lane_split(ds_domain* d, int mode) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    if (mode < 0 || mode > 4) return fail(DS_INVALID_ARGUMENT, "lane split mode is 0..4");
    std::lock_guard<std::mutex> g(d->mu);
    d->lane_split = mode;
    return d->running ? push_control(d) : DS_OK;
}

int ds_tenant_abandonable(ds_domain* d, int tenant, int enable) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    if (tenant < 0 || tenant >= (int)d->tenants.size()) return fail(DS_INVALID_ARGUMENT, "unknown tenant");
    std::lock_guard<std::mutex> g(d->mu);
    if (d->running) return fail(DS_ALREADY_RUNNING, "set before ds_start");
    if (enable) d->retry_mask |= 1ull << tenant;
    else d->retry_mask &= ~(1ull << tenant);
    return DS_OK;
}

int ds_set_lend(ds_domain* d, int lend_tenant) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> g(d->mu);
    d->lend_tenant = lend_tenant;
    return push_control(d);
}

// bind (types.cpp:62-74): BindConflict if the pctx is bound, DoubleBind if the
// tenant is mapped; spatial feasibility (sum of bound tiers <= 1, engine.cpp:721-725)
int ds_bind(ds_domain* d, int tenant, int pctx) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> g(d->mu);
    if (tenant < 0 || tenant >= (int)d->tenants.size()) return fail(DS_INVALID_ARGUMENT, "unknown tenant");
    if (pctx < 0 || pctx >= (int)d->pctxs.size()) return fail(DS_INVALID_ARGUMENT, "unknown pctx");
    Pctx& p = d->pctxs[pctx];
    if (p.bound >= 0) return fail(DS_BIND_CONFLICT, "pctx " + std::to_string(pctx) + " is bound");
    if (d->tenants[tenant]->bound_pctx >= 0) return fail(DS_DOUBLE_BIND, "vctx " + std::to_string(tenant) + " is mapped");
    // exact rational feasibility: sum(num_i/den_i) + p <= 1
    long double sum = (long double)p.num / p.den;
    for (const Pctx& q : d->pctxs)
        if (q.bound >= 0) sum += (long double)q.num / q.den;
    if (sum > 1.0L + 1e-12L) return fail(DS_CONFIG_ERROR, "bind violates spatial feasibility");
    std::vector<int> slots = pick_slots(d, p.n_sms);
    if ((int)slots.size() < p.n_sms) return fail(DS_CONFIG_ERROR, "not enough free SMs");
    for (int s : slots) d->owner[s] = tenant;
    p.slots = slots;
    p.bound = tenant;
    d->tenants[tenant]->bound_pctx = pctx;
    return push_control(d);
}

static int unbind_locked(ds_domain* d, int tenant) {
    int pc = d->tenants[tenant]->bound_pctx;
    if (pc < 0) return fail(DS_BIND_CONFLICT, "unbind of a pair that is not bound");  // types.cpp:77-78
    Pctx& p = d->pctxs[pc];
    for (int s : p.slots) d->owner[s] = -1;
    p.slots.clear();
    p.bound = -1;
    d->tenants[tenant]->bound_pctx = -1;
    return DS_OK;
}

int ds_unbind(ds_domain* d, int tenant) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> g(d->mu);
    if (tenant < 0 || tenant >= (int)d->tenants.size()) return fail(DS_INVALID_ARGUMENT, "unknown tenant");
    int st = unbind_locked(d, tenant);
    if (st) return st;
    return push_control(d);
}

// begin_migration (engine.cpp:620-672) on one GPU: unbind + bind in one
// control-word change; SMs leaving the tenant yield at their block boundary.
int ds_migrate(ds_domain* d, int tenant, int dst) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> g(d->mu);
    if (tenant < 0 || tenant >= (int)d->tenants.size()) return fail(DS_INVALID_ARGUMENT, "unknown tenant");
    if (dst < 0 || dst >= (int)d->pctxs.size()) return fail(DS_INVALID_ARGUMENT, "unknown pctx");
    Pctx& p = d->pctxs[dst];
    if (p.bound >= 0) return fail(DS_BIND_CONFLICT, "remap to a bound pctx");
    int src = d->tenants[tenant]->bound_pctx;
    long double sum = (long double)p.num / p.den;
    for (int i = 0; i < (int)d->pctxs.size(); ++i)
        if (d->pctxs[i].bound >= 0 && i != src) sum += (long double)d->pctxs[i].num / d->pctxs[i].den;
    if (sum > 1.0L + 1e-12L) return fail(DS_CONFIG_ERROR, "remap violates spatial feasibility");
    std::vector<int> keep;
    if (src >= 0) {
        keep = d->pctxs[src].slots;
        unbind_locked(d, tenant);
    }
    // prefer SMs the tenant already holds (no yield needed there)
    std::vector<int> slots;
    for (int s : keep)
        if ((int)slots.size() < p.n_sms) slots.push_back(s);
    for (int s : slots) d->owner[s] = tenant;
    if ((int)slots.size() < p.n_sms) {
        std::vector<int> more = pick_slots(d, p.n_sms - (int)slots.size());
        for (int s : more) {
            d->owner[s] = tenant;
            slots.push_back(s);
        }
    }
    if ((int)slots.size() < p.n_sms) return fail(DS_CONFIG_ERROR, "not enough free SMs");
    p.slots = slots;
    p.bound = tenant;
    d->tenants[tenant]->bound_pctx = dst;
    return push_control(d);
}

// signal_preempt (engine.cpp:756-806): the bound tenant loses the pctx's SMs
// at its next logical-block boundary; its launch stays paused in its claim word.
int ds_preempt(ds_domain* d, int pctx) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> g(d->mu);
    if (pctx < 0 || pctx >= (int)d->pctxs.size()) return fail(DS_INVALID_ARGUMENT, "unknown pctx");
    Pctx& p = d->pctxs[pctx];
    if (p.bound < 0) return DS_OK;  // preempting an unbound pctx is a no-op (engine.cpp:738-746)
    unbind_locked(d, p.bound);
    return push_control(d);
}

int ds_bound_pctx(ds_domain* d, int tenant, int* pctx) {
    if (check_dom(d) || !pctx) return fail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(d->mu);
    if (tenant < 0 || tenant >= (int)d->tenants.size()) return fail(DS_INVALID_ARGUMENT, "unknown tenant");
    *pctx = d->tenants[tenant]->bound_pctx;
    return DS_OK;
}

int ds_quota_at_claim(ds_domain* d, int tenant, uint64_t seq, uint32_t block, const int32_t* owner,
                      const int32_t* lender, int n) {
    if (check_dom(d) || n != d->num_sms) return fail(DS_INVALID_ARGUMENT, "control word needs num_sms entries");
    std::lock_guard<std::mutex> g(d->mu);
    if (d->n_triggers >= ds::kMaxTriggers) return fail(DS_CONFIG_ERROR, "trigger table full");
    std::vector<ds::ClaimTrigger> one(1);
    ds::ClaimTrigger& tr = one[0];
    tr.tenant = tenant;
    tr.seq = (uint32_t)seq;
    tr.block = block;
    for (int i = 0; i < DS_MAX_SMS; ++i) {
        tr.owner[i] = -1;
        tr.lender[i] = -1;
    }
    for (int s = 0; s < n; ++s) {
        tr.owner[d->smids[s]] = owner ? owner[s] : -1;
        tr.lender[d->smids[s]] = lender ? lender[s] : -1;
    }
    cudaSetDevice(d->device);
    DS_CUDA(cudaMemcpyAsync(d->d_triggers + d->n_triggers, &tr, sizeof(tr), cudaMemcpyHostToDevice, d->copy_stream));
    d->n_triggers++;
    if (!d->running) d->prestart_triggers = d->n_triggers;
    uint32_t cnt = (uint32_t)d->n_triggers;
    DS_CUDA(cudaMemcpyAsync(&d->d_state->trig_count, &cnt, sizeof(cnt), cudaMemcpyHostToDevice, d->copy_stream));
    DS_CUDA(cudaStreamSynchronize(d->copy_stream));
    // the host mirror follows the last installed trigger (a trigger armed
    // before ds_start leaves the mirror — the control word at launch — alone)
    if (d->running)
    for (int s = 0; s < n; ++s) {
        d->owner[s] = owner ? owner[s] : -1;
        d->lender[s] = lender ? lender[s] : -1;
    }
    return DS_OK;
}

int ds_quota_periodic(ds_domain* d, uint64_t period_ns, const int32_t* oa, const int32_t* la, const int32_t* ob,
                      const int32_t* lb, int n) {
    if (check_dom(d) || n != d->num_sms) return fail(DS_INVALID_ARGUMENT, "control word needs num_sms entries");
    std::lock_guard<std::mutex> g(d->mu);
    for (int i = 0; i < DS_MAX_SMS; ++i)
        for (int k = 0; k < 2; ++k) {
            d->mb->per_owner[k][i] = -1;
            d->mb->per_lender[k][i] = -1;
        }
    for (int s = 0; s < n; ++s) {
        int sm = d->smids[s];
        d->mb->per_owner[0][sm] = oa ? oa[s] : -1;
        d->mb->per_lender[0][sm] = la ? la[s] : -1;
        d->mb->per_owner[1][sm] = ob ? ob[s] : -1;
        d->mb->per_lender[1][sm] = lb ? lb[s] : -1;
    }
    d->mb->periodic_ns = period_ns;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    d->mb->hot[ds::kHotPGen] = d->mb->hot[ds::kHotPGen] + 1;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    return DS_OK;
}

// Host -> device control round trip: write a control word, spin until the
// loader acknowledges it installed (host-mapped ack), n times; ns per sample.
int ds_ctl_roundtrip(ds_domain* d, int n, uint64_t* out_ns) {
    if (check_dom(d) || !out_ns) return fail(DS_INVALID_ARGUMENT, "null");
    if (!d->running) return fail(DS_NOT_RUNNING, "executor not running");
    for (int i = 0; i < n; ++i) {
        uint32_t want;
        auto t0 = std::chrono::steady_clock::now();
        {
            std::lock_guard<std::mutex> g(d->mu);
            push_control(d);
            want = d->mb->hot[ds::kHotGen];
        }
        while (d->mb->ack_gen != want) {
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(5)) return fail(DS_TIMEOUT, "no ack");
        }
        out_ns[i] = (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    }
    return DS_OK;
}

int ds_stats_get(ds_domain* d, ds_stats* out) {
    if (check_dom(d) || !out) return fail(DS_INVALID_ARGUMENT, "null");
    std::memset(out, 0, sizeof(*out));
    out->launches_enqueued = d->enqueued;
    out->launches_completed = d->completed_total.load();
    out->num_sms = d->num_sms;
    out->running = d->running ? 1 : 0;
    cudaSetDevice(d->device);
    unsigned long long v[5] = {0, 0, 0, 0, 0};
    DS_CUDA(cudaMemcpyAsync(&v[0], &d->d_state->blocks_executed, 8, cudaMemcpyDeviceToHost, d->copy_stream));
    DS_CUDA(cudaMemcpyAsync(&v[1], &d->d_state->ctl.gen, 4, cudaMemcpyDeviceToHost, d->copy_stream));
    DS_CUDA(cudaMemcpyAsync(&v[2], &d->d_state->slog_count, 8, cudaMemcpyDeviceToHost, d->copy_stream));
    DS_CUDA(cudaMemcpyAsync(&v[3], &d->d_state->blog_count, 8, cudaMemcpyDeviceToHost, d->copy_stream));
    DS_CUDA(cudaStreamSynchronize(d->copy_stream));
    out->blocks_executed = v[0];
    out->ctl_changes = v[1] & 0xffffffffu;
    out->switches = v[2];
    out->block_log_entries = std::min<uint64_t>(v[3], d->blog_cap);
    out->block_log_dropped = v[3] > d->blog_cap ? v[3] - d->blog_cap : 0;
    return DS_OK;
}

int ds_ledger_get(ds_domain* d, ds_ledger* out) {
    if (check_dom(d) || !out) return fail(DS_INVALID_ARGUMENT, "null");
    std::memset(out, 0, sizeof(*out));
    cudaSetDevice(d->device);
    unsigned long long v[6] = {0, 0, 0, 0, 0, 0};
    DS_CUDA(cudaMemcpyAsync(v, &d->d_state->led_switches, sizeof(v), cudaMemcpyDeviceToHost, d->copy_stream));
    DS_CUDA(cudaStreamSynchronize(d->copy_stream));
    out->ctx_switches = v[0];
    out->ctx_switch_total_ns = v[1];
    out->preemptions = v[2];
    out->preempt_total_ns = v[3];
    out->migrations = v[4];
    out->migration_total_ns = v[5];
    return DS_OK;
}

int ds_kernel_info_get(ds_domain* d, int kernel_id, ds_kernel_info* out) {
    if (check_dom(d) || !out) return fail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(d->mu);
    if (kernel_id < 0 || kernel_id >= (int)d->kernels.size()) return fail(DS_INVALID_ARGUMENT, "unknown kernel");
    const KernelRecord& k = d->kernels[kernel_id];
    out->fingerprint = k.fingerprint;
    out->args_device = k.args_dev;
    out->args_size = (uint32_t)k.args_host.size();
    out->grid = k.gx * k.gy * k.gz;
    out->body = k.body;
    out->phase = k.phase;
    return DS_OK;
}

// Kernel records are immutable (engine.cpp:183-187, 1379-1383): recompute each
// fingerprint from the argument block the executor actually reads (device copy).
int ds_verify_kernels(ds_domain* d, int* first_bad) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> g(d->mu);
    if (first_bad) *first_bad = -1;
    if (d->args_used == 0) return DS_OK;
    std::vector<uint8_t> arena(d->args_used);
    cudaSetDevice(d->device);
    DS_CUDA(cudaMemcpyAsync(arena.data(), d->d_args, d->args_used, cudaMemcpyDeviceToHost, d->copy_stream));
    DS_CUDA(cudaStreamSynchronize(d->copy_stream));
    for (size_t i = 0; i < d->kernels.size(); ++i) {
        const KernelRecord& k = d->kernels[i];
        const uint8_t* dev = arena.data() + (k.args_dev - (uint64_t)d->d_args);
        if (kernel_fingerprint(k, dev) != k.fingerprint) {
            if (first_bad) *first_bad = (int)i;
            return fail(DS_RECORD_MUTATED, "kernel record " + std::to_string(i) + " (" + k.semantic_id +
                                               ") mutated during the run");
        }
    }
    return DS_OK;
}

// vctx_transcripts (engine.hpp:124): executed signatures of completed launches
int ds_transcript(ds_domain* d, int tenant, int32_t* kernel_ids, uint32_t* grids, int cap, int* n) {
    if (check_dom(d) || !n) return fail(DS_INVALID_ARGUMENT, "null");
    if (tenant < 0 || tenant >= (int)d->tenants.size()) return fail(DS_INVALID_ARGUMENT, "unknown tenant");
    std::lock_guard<std::mutex> g(d->mu);
    TenantRecord* t = d->tenants[tenant];
    uint64_t done = t->completed.load();
    int m = (int)std::min<uint64_t>(done, (uint64_t)cap);
    for (int i = 0; i < m; ++i) {
        if (kernel_ids) kernel_ids[i] = t->launched_kernel[i];
        if (grids) grids[i] = t->launched_grid[i];
    }
    *n = (int)done;
    return DS_OK;
}

int ds_logical_progress(ds_domain* d, int tenant, int64_t* out) {
    if (check_dom(d) || !out) return fail(DS_INVALID_ARGUMENT, "null");
    if (tenant < 0 || tenant >= (int)d->tenants.size()) return fail(DS_INVALID_ARGUMENT, "unknown tenant");
    *out = (int64_t)d->tenants[tenant]->completed.load();  // types.hpp:86 logical_progress
    return DS_OK;
}

}  // extern "C"

template <class T>
static int copy_log(ds_domain* d, T* dev, unsigned long long* dcount, uint64_t cap_dev, T* out, int64_t cap,
                    int64_t* n) {
    cudaSetDevice(d->device);
    unsigned long long cnt = 0;
    DS_CUDA(cudaMemcpyAsync(&cnt, dcount, 8, cudaMemcpyDeviceToHost, d->copy_stream));
    DS_CUDA(cudaStreamSynchronize(d->copy_stream));
    uint64_t avail = std::min<uint64_t>(cnt, cap_dev);
    uint64_t m = std::min<uint64_t>(avail, cap < 0 ? 0 : (uint64_t)cap);
    if (m && out) {
        DS_CUDA(cudaMemcpyAsync(out, dev, m * sizeof(T), cudaMemcpyDeviceToHost, d->copy_stream));
        DS_CUDA(cudaStreamSynchronize(d->copy_stream));
    }
    *n = (int64_t)avail;
    return DS_OK;
}

extern "C" {

int ds_block_log(ds_domain* d, ds_block_record* out, int64_t cap, int64_t* n) {
    if (check_dom(d) || !n) return fail(DS_INVALID_ARGUMENT, "null");
    if (!d->d_blog) {
        *n = 0;
        return DS_OK;
    }
    return copy_log(d, d->d_blog, &d->d_state->blog_count, d->blog_cap, out, cap, n);
}

int ds_switch_log(ds_domain* d, ds_switch_record* out, int64_t cap, int64_t* n) {
    if (check_dom(d) || !n) return fail(DS_INVALID_ARGUMENT, "null");
    return copy_log(d, d->d_slog, &d->d_state->slog_count, d->slog_cap, out, cap, n);
}

int ds_ctl_log(ds_domain* d, ds_ctl_record* out, int64_t cap, int64_t* n) {
    if (check_dom(d) || !n) return fail(DS_INVALID_ARGUMENT, "null");
    return copy_log(d, d->d_clog, &d->d_state->clog_count, d->clog_cap, out, cap, n);
}

// Empty the claim-trigger table (all installed triggers must have fired or
// belong to launches that will not run again): triggers fire in install order.
int ds_quota_triggers_reset(ds_domain* d) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> g(d->mu);
    cudaSetDevice(d->device);
    uint32_t z[2] = {0, 0};  // trig_next, trig_count (adjacent)
    DS_CUDA(cudaMemcpyAsync(&d->d_state->trig_next, z, sizeof(z), cudaMemcpyHostToDevice, d->copy_stream));
    DS_CUDA(cudaStreamSynchronize(d->copy_stream));
    d->n_triggers = 0;
    d->prestart_triggers = 0;
    return DS_OK;
}

int ds_clear_logs(ds_domain* d) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    cudaSetDevice(d->device);
    unsigned long long z = 0;
    DS_CUDA(cudaMemcpyAsync(&d->d_state->blog_count, &z, 8, cudaMemcpyHostToDevice, d->copy_stream));
    DS_CUDA(cudaMemcpyAsync(&d->d_state->slog_count, &z, 8, cudaMemcpyHostToDevice, d->copy_stream));
    DS_CUDA(cudaMemcpyAsync(&d->d_state->clog_count, &z, 8, cudaMemcpyHostToDevice, d->copy_stream));
    DS_CUDA(cudaStreamSynchronize(d->copy_stream));
    return DS_OK;
}

int ds_globaltimer(ds_domain* d, uint64_t* ns) {
    if (check_dom(d) || !ns) return fail(DS_INVALID_ARGUMENT, "null");
    cudaSetDevice(d->device);
    // 1 CTA of 32 threads with no smem co-resides with the executor; buffers
    // are preallocated (cudaFree would synchronize with the resident executor)
    ds_dev_probe(1, d->d_probe, d->d_probe + 1, d->d_probe_t, d->copy_stream);
    cudaMemcpyAsync(ns, d->d_probe_t, 8, cudaMemcpyDeviceToHost, d->copy_stream);
    cudaError_t e = cudaStreamSynchronize(d->copy_stream);
    if (e != cudaSuccess) return fail(DS_CUDA_ERROR, cudaGetErrorString(e));
    return DS_OK;
}


// Debug snapshot of the device control state (readable while the executor runs).
int ds_debug_dump(ds_domain* d, char* out, int64_t cap) {
    if (check_dom(d) || !out) return fail(DS_INVALID_ARGUMENT, "null");
    cudaSetDevice(d->device);
    std::vector<uint8_t> buf(sizeof(ds::DevState));
    DS_CUDA(cudaMemcpyAsync(buf.data(), d->d_state, sizeof(ds::DevState), cudaMemcpyDeviceToHost, d->copy_stream));
    DS_CUDA(cudaStreamSynchronize(d->copy_stream));
    const ds::DevState* st = reinterpret_cast<const ds::DevState*>(buf.data());
    std::string s;
    char line[256];
    snprintf(line, sizeof line, "ctl.gen=%u exit=%u blocks=%llu comp=%llu trig_next=%u trig_count=%u mb.gen=%u host_comp_next=%llu\n",
             st->ctl.gen, st->ctl.exit, st->blocks_executed, st->completion_count, st->trig_next, st->trig_count,
             d->mb->hot[ds::kHotGen], (unsigned long long)d->comp_next);
    s += line;
    for (int t = 0; t < (int)d->tenants.size(); ++t) {
        const ds::DevTenant& T = st->tenants[t];
        snprintf(line, sizeof line, "tenant %d: claim seq=%u blk=%u tail=%u head=%u host_tail=%u next_seq=%llu completed=%llu\n", t,
                 (unsigned)(T.claim >> 32), (unsigned)(T.claim & 0xffffffffu), T.tail, T.head, d->mb->hot[ds::kHotTail + t],
                 (unsigned long long)d->tenants[t]->next_seq, (unsigned long long)d->tenants[t]->completed.load());
        s += line;
    }
    int owned = 0, lent = 0;
    for (int i = 0; i < DS_MAX_SMS; ++i) {
        owned += (int32_t)(uint32_t)st->ctl.word[i] >= 0;
        lent += (int32_t)(uint32_t)(st->ctl.word[i] >> 32) >= 0;
    }
    snprintf(line, sizeof line, "device ctl: %d SMs owned, %d with lender\n", owned, lent);
    s += line;
    if ((int64_t)s.size() + 1 > cap) s.resize(cap - 1);
    std::memcpy(out, s.c_str(), s.size() + 1);
    return DS_OK;
}

// ---- TMA tensor maps (host encode through the driver entry point; libcuda is
// never linked, so the library still loads on a CPU-only host) ----
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int ds_tensor_map_bf16_2d(void* out128, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                          uint32_t box_cols) {
    return ds_tensor_map_bf16_2d_pitched(out128, base, rows, cols, cols, box_rows, box_cols);
}

// rows x cols valid elements of a row-major bf16 array whose rows are `pitch`
// elements apart (cols <= pitch): boxes reaching past the valid extent are
// zero-filled by the TMA unit and never read from memory; stores past it are
// clipped (the GEMM tenant on unpadded shapes, e.g. conv1's K = 147)
int ds_tensor_map_bf16_2d_pitched(void* out128, const void* base, uint64_t rows, uint64_t cols, uint64_t pitch,
                                  uint32_t box_rows, uint32_t box_cols) {
    if (!out128 || !base) return fail(DS_INVALID_ARGUMENT, "null");
    if (cols == 0 || rows == 0 || cols > pitch) return fail(DS_INVALID_ARGUMENT, "need 0 < cols <= pitch, rows > 0");
    if (box_cols * 2 != 128 && box_cols * 2 != 64)
        return fail(DS_CONFIG_ERROR, "box inner extent must be 128 B (SWIZZLE_128B) or 64 B (SWIZZLE_64B)");
    if ((pitch * 2) % 16 != 0 || ((uintptr_t)base & 15)) return fail(DS_CONFIG_ERROR, "row pitch / base must be 16-B aligned");
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            return fail(DS_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        fn = (EncodeTiledFn)p;
    }
    CUtensorMap m;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {pitch * 2};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, box_cols * 2 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(DS_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    std::memcpy(out128, &m, 128);
    return DS_OK;
}

// KV-cache view for the attention body: [rows][128] bf16 as a 3-D tensor
// {64 dims, rows, 2 halves} (strides 256 B per row, 128 B per half); one box
// {64, box_rows, 2} lands as two half-tiles [box_rows][64] (128-B rows,
// SWIZZLE_128B), dims 0-63 then 64-127: one smem row per KV position, so the
// body's ldmatrix reads are conflict-free, and one TMA per chunk operand.
int ds_tensor_map_bf16_kv(void* out128, const void* base, uint64_t rows, uint32_t box_rows) {
    if (!out128 || !base) return fail(DS_INVALID_ARGUMENT, "null");
    if (((uintptr_t)base & 15)) return fail(DS_CONFIG_ERROR, "base must be 16-B aligned");
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            return fail(DS_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        fn = (EncodeTiledFn)p;
    }
    CUtensorMap m;
    if ((int)box_rows != ds_attn_chunk()) return fail(DS_CONFIG_ERROR, "kv box rows must equal ds_attn_chunk()");
    cuuint64_t dims[3] = {64, rows, 2};
    cuuint64_t strides[2] = {256, 128};
    cuuint32_t box[3] = {64, box_rows, 2};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(DS_CUDA_ERROR, "cuTensorMapEncodeTiled(kv) failed (" + std::to_string((int)r) + ")");
    std::memcpy(out128, &m, 128);
    return DS_OK;
}

extern "C" cudaError_t ds_dev_solo_trace(void* buf);
// per-CTA stamps of plain-grid solo launches into dev_buf (u64 [grid][4]:
// entry, TMEM allocated, body returned, exit); nullptr turns them off
int ds_solo_trace(int device, void* dev_buf) {
    if (cudaSetDevice(device) != cudaSuccess) return fail(DS_CUDA_ERROR, "cudaSetDevice");
    cudaError_t e = ds_dev_solo_trace(dev_buf);
    if (e != cudaSuccess) return fail(DS_CUDA_ERROR, cudaGetErrorString(e));
    return DS_OK;
}

int ds_solo_launch(int device, const ds_kernel_desc* k, void* stream) {
    if (!k) return fail(DS_INVALID_ARGUMENT, "null desc");
    if (k->body <= DS_BODY_NONE || k->body >= DS_BODY_COUNT) return fail(DS_CONFIG_ERROR, "unknown body");
    if (k->args_size > ds::kMaxArgs) return fail(DS_CONFIG_ERROR, "args too large");
    cudaSetDevice(device);
    cudaStream_t s = (cudaStream_t)stream;
    void* dargs = nullptr;
    DS_CUDA(cudaMalloc(&dargs, ds::kMaxArgs));
    DS_CUDA(cudaMemcpyAsync(dargs, k->args, k->args_size, cudaMemcpyHostToDevice, s));
    uint32_t smem = ds_dev_body_smem(k->body);
    cudaError_t e = ds_dev_launch_solo(k->body, dargs, k->grid_x, k->grid_y, k->grid_z, smem, s);
    cudaStreamSynchronize(s);
    cudaFree(dargs);
    if (e != cudaSuccess) return fail(DS_CUDA_ERROR, std::string("solo launch: ") + cudaGetErrorString(e));
    return DS_OK;
}

int ds_solo_launch_registered(ds_domain* d, int kernel_id, void* stream) {
    if (check_dom(d)) return DS_INVALID_ARGUMENT;
    if (kernel_id < 0 || kernel_id >= (int)d->kernels.size()) return fail(DS_INVALID_ARGUMENT, "unknown kernel");
    const KernelRecord& k = d->kernels[kernel_id];
    cudaSetDevice(d->device);
    cudaError_t e = ds_dev_launch_solo(k.body, (const void*)k.args_dev, k.gx, k.gy, k.gz, ds_dev_body_smem(k.body),
                                       (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(DS_CUDA_ERROR, std::string("solo launch: ") + cudaGetErrorString(e));
    return DS_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Peer memory for the DP all-reduce body (bodies/collective.cuh)
// ---------------------------------------------------------------------------
extern "C" {

int ds_ipc_alloc(int device, uint64_t bytes, void** ptr) {
    if (!ptr || bytes == 0) return fail(DS_INVALID_ARGUMENT, "null / empty");
    if (cudaSetDevice(device) != cudaSuccess) return fail(DS_NO_DEVICE, "bad device ordinal");
    if (cudaMalloc(ptr, bytes) != cudaSuccess) return fail(DS_CUDA_ERROR, "cudaMalloc");
    if (cudaMemset(*ptr, 0, bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
        return fail(DS_CUDA_ERROR, "cudaMemset");
    return DS_OK;
}

int ds_ipc_free(int device, void* ptr) {
    if (cudaSetDevice(device) != cudaSuccess) return fail(DS_NO_DEVICE, "bad device ordinal");
    return cudaFree(ptr) == cudaSuccess ? DS_OK : fail(DS_CUDA_ERROR, "cudaFree");
}

int ds_ipc_handle(void* ptr, void* handle64) {
    if (!ptr || !handle64) return fail(DS_INVALID_ARGUMENT, "null");
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, ptr) != cudaSuccess) return fail(DS_CUDA_ERROR, "cudaIpcGetMemHandle");
    static_assert(sizeof(h) == 64, "IPC handle is 64 bytes");
    std::memcpy(handle64, &h, 64);
    return DS_OK;
}

int ds_ipc_open(int device, const void* handle64, void** ptr) {
    if (!ptr || !handle64) return fail(DS_INVALID_ARGUMENT, "null");
    if (cudaSetDevice(device) != cudaSuccess) return fail(DS_NO_DEVICE, "bad device ordinal");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    if (cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
        return fail(DS_CUDA_ERROR, "cudaIpcOpenMemHandle");
    return DS_OK;
}

extern "C" cudaError_t ds_dev_ffma_probe(int nblocks, int iters, float* out, cudaStream_t s);

int ds_measure_ffma_peak(int device, double* tflops) {
    if (!tflops) return fail(DS_INVALID_ARGUMENT, "null");
    if (cudaSetDevice(device) != cudaSuccess) return fail(DS_NO_DEVICE, "bad device ordinal");
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    float* out = nullptr;
    DS_CUDA(cudaMalloc(&out, 4 * 4096));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = 4 * nsm, iters = 4096;
    double best = 0.0;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0, 0);
        cudaError_t e = ds_dev_ffma_probe(blocks, iters, out, 0);
        cudaEventRecord(e1, 0);
        if (e != cudaSuccess || cudaEventSynchronize(e1) != cudaSuccess) {
            cudaFree(out);
            return fail(DS_CUDA_ERROR, "ffma probe failed");
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flop = 2.0 * 8 * 16 * (double)iters * 256.0 * blocks;
        if (rep > 0 && ms > 0.f) best = std::max(best, flop / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    *tflops = best;
    return DS_OK;
}

int ds_dp_abort(int device, void* flags) {
    if (!flags) return fail(DS_INVALID_ARGUMENT, "null");
    if (cudaSetDevice(device) != cudaSuccess) return fail(DS_NO_DEVICE, "bad device ordinal");
    const unsigned long long one = 1;
    // a copy-engine write: works while the resident executor holds every SM
    if (cudaMemcpy(static_cast<unsigned long long*>(flags) + 2 * 64, &one, 8, cudaMemcpyHostToDevice) != cudaSuccess)
        return fail(DS_CUDA_ERROR, "cudaMemcpy");
    return DS_OK;
}

int ds_ipc_close(int device, void* ptr) {
    if (cudaSetDevice(device) != cudaSuccess) return fail(DS_NO_DEVICE, "bad device ordinal");
    return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? DS_OK : fail(DS_CUDA_ERROR, "cudaIpcCloseMemHandle");
}

}  // extern "C"
