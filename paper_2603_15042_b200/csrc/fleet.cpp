// Fleet — the cross-device layer over per-GPU domains:
// global exceptions with emergency migration to a standby device, and
// working-set tracking with eager / lazy copies and demand faults for
// planned cross-device migrations.  Each GPU stays an independent sharing
// domain (own executor, arbiter, pctx pool); the fleet moves a job (one
// tenant per device it has lived on) between them.
//
//   apply_global_exception  proj/src/engine/engine.cpp:1095-1122 -> ds_fleet_global_exception
//   emergency_migrate       engine.cpp:1124-1166                  -> emergency_target / ds_emergency_target
//   begin_migration         engine.cpp:620-672                    -> begin_migration()
//   on_migration_done       engine.cpp:986-1009                   -> eager copy complete, regions resident
//   advance_lazy            engine.cpp:596-618                    -> advance_lazy() (copy-stream events)
//   service_demand_faults   engine.cpp:563-594                    -> service_demand_faults() at launch
//   finish_run (regions)    engine.cpp:861-866                    -> touched regions dirty, resident on dev
//
// B200 realisation: a job's regions are device buffers; a move copies them
// peer to peer on the copy engines (cudaMemcpyPeerAsync, no SMs) and
// re-registers the job's kernels on the destination with their pointer
// arguments relocated (ds_reloc).  A launch interrupted by a global
// exception resumes on the standby at its next unclaimed logical block
// (ds_launch_from): every block runs exactly once, so results are
// bit-identical to an uninterrupted run ("kernel resumes, never restarts").
// Differences from the simulator, by construction of real hardware: regions
// start resident where the caller allocated them (the reference starts with
// none resident and pays a cold copy at the first bind), copy time is
// measured instead of bytes / copy_bandwidth, and the jobs of a failed
// device are drained together and then moved in pool order (the reference
// moves a running vctx at its own boundary event).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/detshare/ds.h"

namespace {

thread_local std::string f_last_error;
int ffail(int st, const std::string& w) {
    f_last_error = w;
    return st;
}

int64_t now_ns() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

// a/b >= c/d for positive denominators
bool frac_ge(int64_t a, int64_t b, int64_t c, int64_t d) { return (__int128)a * d >= (__int128)c * b; }
bool frac_lt(int64_t a, int64_t b, int64_t c, int64_t d) { return (__int128)a * d < (__int128)c * b; }
bool frac_gt(int64_t a, int64_t b, int64_t c, int64_t d) { return (__int128)a * d > (__int128)c * b; }

}  // namespace

struct Frac_t {
    int64_t num, den;
};

extern "C" {

const char* ds_fleet_last_error(void) { return f_last_error.c_str(); }

// emergency_migrate's target rule (engine.cpp:1128-1154): the first healthy
// standby device, in device order, with an unbound pctx that keeps the
// device feasible (sum of bound tiers + tier <= 1); on it the smallest tier
// >= the vctx's current tier, else the largest smaller one (first in pool
// order on ties).  -1: stranded.
int ds_emergency_target(const int32_t* dev_failed, const int32_t* dev_standby, int n_devices,
                        const ds_place_pctx* pctxs, int n_pctxs, int64_t cur_num, int64_t cur_den, int* target) {
    if (!target || n_devices < 0 || n_pctxs < 0 || (n_devices && (!dev_failed || !dev_standby)) ||
        (n_pctxs && !pctxs) || cur_den <= 0)
        return ffail(DS_INVALID_ARGUMENT, "bad arguments");
    *target = -1;
    for (int dv = 0; dv < n_devices; ++dv) {
        if (dev_failed[dv] || !dev_standby[dv]) continue;
        // bound tier sum of the device as an exact fraction over a common den
        __int128 sn = 0, sd = 1;
        for (int i = 0; i < n_pctxs; ++i) {
            const ds_place_pctx& p = pctxs[i];
            if (p.device != dv || !p.bound) continue;
            sn = sn * p.tier_den + (__int128)p.tier_num * sd;
            sd = sd * p.tier_den;
            // keep small: tiers have small denominators
            __int128 a = sn < 0 ? -sn : sn, b = sd;
            while (b) {
                __int128 t = a % b;
                a = b;
                b = t;
            }
            if (a > 1) {
                sn /= a;
                sd /= a;
            }
        }
        int above = -1, below = -1;
        for (int i = 0; i < n_pctxs; ++i) {
            const ds_place_pctx& p = pctxs[i];
            if (p.device != dv || p.bound || p.tier_den <= 0) continue;
            // sum + tier > 1 ?
            if (sn * p.tier_den + (__int128)p.tier_num * sd > sd * p.tier_den) continue;
            if (frac_ge(p.tier_num, p.tier_den, cur_num, cur_den)) {
                if (above < 0 || frac_lt(p.tier_num, p.tier_den, pctxs[above].tier_num, pctxs[above].tier_den))
                    above = i;
            } else if (below < 0 || frac_gt(p.tier_num, p.tier_den, pctxs[below].tier_num, pctxs[below].tier_den)) {
                below = i;
            }
        }
        const int chosen = above >= 0 ? above : below;
        if (chosen >= 0) {
            *target = chosen;
            return DS_OK;
        }
    }
    return DS_OK;
}

}  // extern "C"

struct ds_fleet {
    struct Device {
        ds_domain* dom = nullptr;
        int cuda = 0;
        bool standby = false;
        bool failed = false;
        cudaStream_t copy = nullptr;  // eager copies and demand faults (copy engines)
        cudaStream_t lazy = nullptr;  // background (lazy) copies into this device
    };
    struct Region {
        uint64_t bytes = 0;
        bool dirty = false;
        uint64_t resident = 0;        // bit d: an up-to-date copy lives on device d
        std::vector<void*> ptr;       // per device (nullptr: never allocated there)
        std::vector<bool> owned;      // allocated by the fleet (freed at destroy)
        int lazy_dst = -1;            // a background copy into lazy_dst is in flight
        cudaEvent_t lazy_ev = nullptr;
        int64_t lazy_issued = 0;
    };
    struct Kernel {
        std::string semantic_id;
        ds_kernel_desc desc{};
        std::vector<uint8_t> args;
        std::vector<ds_reloc> relocs;
        std::vector<int32_t> touched;
        std::vector<int> on_dev;      // registered kernel id per device (-1)
    };
    struct Launch {
        int kernel = -1;
        int dev = -1;
        uint64_t dseq = 0;            // device launch sequence (valid once issued)
        uint32_t first_block = 0;
        bool issued = false;
    };
    struct Job {
        std::string name;
        int priority = DS_BEST_EFFORT;
        int dev = -1;
        std::vector<int> tenant;      // per device (-1)
        int pctx = -1;                // bound pctx on dev
        int status = 0;               // VctxStatus: 0 Active, 1 Failed, 2 Stranded (types.hpp:77)
        std::vector<Region> regions;
        std::vector<Kernel> kernels;
        std::vector<Launch> launches;
        int active_migration = -1;
    };

    std::vector<Device> devs;
    std::vector<Job> jobs;
    std::vector<ds_migration_info> migrations;
    ds_fleet_ledger ledger{};
    std::mutex mu;

    Device& dev(int d) { return devs[(size_t)d]; }

    int ensure_region_on(Job& j, int r, int d) {
        Region& g = j.regions[(size_t)r];
        if (g.ptr[(size_t)d]) return DS_OK;
        cudaSetDevice(dev(d).cuda);
        void* p = nullptr;
        if (cudaMalloc(&p, g.bytes) != cudaSuccess) return ffail(DS_CUDA_ERROR, "cudaMalloc region");
        g.ptr[(size_t)d] = p;
        g.owned[(size_t)d] = true;
        return DS_OK;
    }

    int copy_region(Job& j, int r, int src, int dst, cudaStream_t s) {
        Region& g = j.regions[(size_t)r];
        const void* sp = g.ptr[(size_t)src];
        void* dp = g.ptr[(size_t)dst];
        uint64_t b = g.bytes;
        return ds_migrate_regions(dev(src).cuda, dev(dst).cuda, &sp, &dp, &b, 1, s);
    }

    // any device holding an up-to-date copy (lowest index)
    int source_of(const Region& g, int not_dev) const {
        for (size_t d = 0; d < devs.size(); ++d)
            if (((g.resident >> d) & 1ull) && (int)d != not_dev && g.ptr[d]) return (int)d;
        return -1;
    }

    // advance_lazy (engine.cpp:596-618): finished background copies land
    void advance_lazy(Job& j) {
        for (Region& g : j.regions) {
            if (g.lazy_dst < 0) continue;
            if (cudaEventQuery(g.lazy_ev) == cudaSuccess) {
                g.resident |= 1ull << g.lazy_dst;
                g.dirty = false;
                g.lazy_dst = -1;
            }
        }
        cudaGetLastError();  // cudaErrorNotReady is not an error here
    }

    void cancel_lazy(Job& j) {
        // a new migration supersedes outstanding transfers (engine.cpp:623)
        for (Region& g : j.regions) {
            if (g.lazy_dst < 0) continue;
            cudaEventSynchronize(g.lazy_ev);  // the bytes are in flight on a copy engine; let them land unused
            g.lazy_dst = -1;
        }
    }

    int register_on(Job& j, int k, int d) {
        Kernel& K = j.kernels[(size_t)k];
        if (K.on_dev[(size_t)d] >= 0) return DS_OK;
        std::vector<uint8_t> a = K.args;
        for (const ds_reloc& rl : K.relocs) {
            const Region& g = j.regions[(size_t)rl.region];
            const uint64_t v = (uint64_t)(uintptr_t)g.ptr[(size_t)d] + rl.region_offset;
            std::memcpy(a.data() + rl.args_offset, &v, 8);
        }
        ds_kernel_desc desc = K.desc;
        desc.semantic_id = K.semantic_id.c_str();
        desc.args = a.empty() ? nullptr : a.data();
        desc.args_size = (uint32_t)a.size();
        int id = -1;
        int st = ds_kernel_register(dev(d).dom, &desc, &id);
        if (st) return st;
        K.on_dev[(size_t)d] = id;
        return DS_OK;
    }

    int ensure_tenant(Job& j, int d) {
        if (j.tenant[(size_t)d] >= 0) return DS_OK;
        ds_tenant_desc td{j.name.c_str(), j.priority};
        int t = -1;
        int st = ds_tenant_register(dev(d).dom, &td, &t);
        if (st) return st;
        j.tenant[(size_t)d] = t;
        return DS_OK;
    }

    bool running(int d) {
        ds_stats s{};
        return ds_stats_get(dev(d).dom, &s) == DS_OK && s.running;
    }

    // one executor per physical GPU at a time: a device whose GPU hosts
    // another fleet device's executor starts only once that one holds no
    // active job (then it is stopped).  Distinct GPUs never interact.
    int ensure_running(int d, const Job* moving) {
        if (running(d)) return DS_OK;
        for (size_t o = 0; o < devs.size(); ++o) {
            if ((int)o == d || devs[o].cuda != dev(d).cuda || !running((int)o)) continue;
            for (const Job& j : jobs)
                if (j.dev == (int)o && j.status == 0 && &j != moving)
                    return ffail(DS_CONFIG_ERROR, "GPU " + std::to_string(dev(d).cuda) +
                                                      " runs another device's executor with active jobs");
            ds_stop(devs[o].dom);
        }
        return ds_start(dev(d).dom);
    }

    // service_demand_faults (engine.cpp:563-594): before a kernel starts on
    // d, every region it touches that is not resident there is brought in
    // now (a lazy copy in flight is waited for; else a synchronous copy)
    int service_demand_faults(Job& j, const Kernel& K, int d, int& faults) {
        advance_lazy(j);
        faults = 0;
        for (int32_t r : K.touched) {
            Region& g = j.regions[(size_t)r];
            if ((g.resident >> d) & 1ull) continue;
            const int64_t t0 = now_ns();
            if (g.lazy_dst == d) {
                cudaEventSynchronize(g.lazy_ev);
                g.lazy_dst = -1;
            } else {
                const int src = source_of(g, d);
                if (src < 0) return ffail(DS_TRACE_VIOLATION, "region has no up-to-date copy");
                int st = ensure_region_on(j, r, d);
                if (st) return st;
                st = copy_region(j, r, src, d, dev(d).copy);
                if (st) return st;
                if (cudaStreamSynchronize(dev(d).copy) != cudaSuccess) return ffail(DS_CUDA_ERROR, "demand copy");
            }
            g.resident |= 1ull << d;
            g.dirty = false;
            ++faults;
            ledger.demand_faults++;
            ledger.demand_fault_total_ns += now_ns() - t0;
        }
        return DS_OK;
    }

    int issue(Job& j, size_t li) {
        Launch& L = j.launches[li];
        Kernel& K = j.kernels[(size_t)L.kernel];
        const int d = j.dev;
        int faults = 0;
        int st = service_demand_faults(j, K, d, faults);
        if (st) return st;
        if (j.active_migration >= 0) migrations[(size_t)j.active_migration].demand_faults += faults;
        if ((st = register_on(j, L.kernel, d))) return st;
        uint64_t seq = 0;
        const int t = j.tenant[(size_t)d];
        st = L.first_block ? ds_launch_from(dev(d).dom, t, K.on_dev[(size_t)d], (uint64_t)li, L.first_block, &seq)
                           : ds_launch(dev(d).dom, t, K.on_dev[(size_t)d], (uint64_t)li, &seq);
        if (st) return st;
        L.dev = d;
        L.dseq = seq;
        L.issued = true;
        // finish_run (engine.cpp:861-866): the kernel's regions are dirty and
        // live on d only (marked at issue: every other copy is stale from now)
        for (int32_t r : K.touched) {
            Region& g = j.regions[(size_t)r];
            g.dirty = true;
            g.resident = 1ull << d;
        }
        return DS_OK;
    }

    Frac_t tier_of(int d, int pctx) {
        Frac_t f{0, 1};
        if (pctx < 0) return f;
        int n = 0, b = -1;
        ds_pctx_info(dev(d).dom, pctx, &f.num, &f.den, &n, &b);
        return f;
    }

    // begin_migration (engine.cpp:620-672) once the job is drained on its
    // source; resume = (launch index, first block) of the first unfinished
    // launch.  The eager set is copied now; the lazy set follows on the
    // destination's lazy stream.
    int begin_migration(Job& j, int ji, int dst, int dst_pctx, bool emergency, size_t resume_li, uint32_t resume_block) {
        const int src = j.dev;
        const int src_pctx = j.pctx;
        const int64_t t0 = now_ns();
        cancel_lazy(j);
        // the whole working set is reserved on the destination up front (no
        // allocation once its executor may be resident)
        for (size_t r = 0; r < j.regions.size(); ++r) {
            int st0 = ensure_region_on(j, (int)r, dst);
            if (st0) return st0;
        }
        std::vector<ds_region> ws(j.regions.size());
        for (size_t r = 0; r < j.regions.size(); ++r) {
            ws[r].id = (int32_t)r;
            ws[r].dirty = j.regions[r].dirty;
            ws[r].bytes = j.regions[r].bytes;
            ws[r].resident_mask = j.regions[r].resident;
        }
        std::vector<int32_t> eager(ws.size()), lazy(ws.size());
        int ne = 0, nl = 0;
        uint64_t eb = 0, lb = 0;
        int st;
        if (emergency) {
            st = ds_full_eager_set(ws.data(), (int)ws.size(), eager.data(), &ne, &eb);
        } else {
            // the migration set follows the job's next kernel (head_kernel)
            std::vector<int32_t> touched;
            if (resume_li < j.launches.size()) touched = j.kernels[(size_t)j.launches[resume_li].kernel].touched;
            st = ds_compute_migration_set(ws.data(), (int)ws.size(), touched.data(), (int)touched.size(), dst,
                                          eager.data(), &ne, &eb, lazy.data(), &nl, &lb);
        }
        if (st) return ffail(st, "migration set");
        // regions dirty only somewhere else than src are copied from there
        for (int i = 0; i < ne; ++i) {
            const int r = eager[(size_t)i];
            if ((st = ensure_region_on(j, r, dst))) return st;
            Region& g = j.regions[(size_t)r];
            if ((g.resident >> dst) & 1ull) continue;
            const int from = ((g.resident >> src) & 1ull) ? src : source_of(g, dst);
            if (from < 0) return ffail(DS_TRACE_VIOLATION, "region has no up-to-date copy");
            if ((st = copy_region(j, r, from, dst, dev(dst).copy))) return st;
        }
        if (cudaStreamSynchronize(dev(dst).copy) != cudaSuccess) return ffail(DS_CUDA_ERROR, "eager copy");
        // on_migration_done (engine.cpp:986-1009): eager regions resident, clean
        for (int i = 0; i < ne; ++i) {
            Region& g = j.regions[(size_t)eager[(size_t)i]];
            g.resident |= 1ull << dst;
            g.dirty = false;
        }
        // lazy set: background copies in region order (the reference's lazy queue)
        for (int i = 0; i < nl; ++i) {
            const int r = lazy[(size_t)i];
            if ((st = ensure_region_on(j, r, dst))) return st;
            Region& g = j.regions[(size_t)r];
            const int from = ((g.resident >> src) & 1ull) ? src : source_of(g, dst);
            if (from < 0) continue;
            if ((st = copy_region(j, r, from, dst, dev(dst).lazy))) return st;
            cudaSetDevice(dev(dst).cuda);
            if (!g.lazy_ev) cudaEventCreateWithFlags(&g.lazy_ev, cudaEventDisableTiming);
            cudaEventRecord(g.lazy_ev, dev(dst).lazy);
            g.lazy_dst = dst;
            g.lazy_issued = now_ns();
        }
        if ((st = ensure_running(dst, &j))) return st;
        if ((st = ensure_tenant(j, dst))) return st;
        j.dev = dst;
        j.pctx = -1;
        if (dst_pctx >= 0) {
            if ((st = ds_bind(dev(dst).dom, j.tenant[(size_t)dst], dst_pctx))) return st;
            j.pctx = dst_pctx;
        }
        ds_migration_info m{};
        m.job = ji;
        m.src_device = src;
        m.src_pctx = src_pctx;
        m.dst_device = dst;
        m.dst_pctx = dst_pctx;
        m.emergency = emergency;
        m.eager_bytes = eb;
        m.lazy_bytes = lb;
        m.start_ns = t0;
        m.resumed_launch = resume_li;
        m.resumed_block = resume_block;
        j.active_migration = (int)migrations.size();
        migrations.push_back(m);
        // the unfinished launches, in program order, the first one from its block
        for (size_t li = resume_li; li < j.launches.size(); ++li) {
            Launch& L = j.launches[li];
            L.issued = false;
            L.first_block = li == resume_li ? resume_block : 0;
            if ((st = issue(j, li))) return st;
        }
        migrations.back().end_ns = now_ns();
        ledger.migrations++;
        if (emergency) ledger.emergency_migrations++;
        ledger.migration_total_ns += migrations.back().end_ns - t0;
        ledger.eager_bytes += eb;
        ledger.lazy_bytes += lb;
        return DS_OK;
    }

    // first unfinished launch of a drained job and its resume block
    int resume_point(Job& j, size_t& li, uint32_t& block) {
        const int d = j.dev;
        const int t = j.tenant[(size_t)d];
        ds_progress p{};
        int st = ds_tenant_progress(dev(d).dom, t, &p);
        if (st) return st;
        li = j.launches.size();
        block = 0;
        for (size_t i = 0; i < j.launches.size(); ++i) {
            const Launch& L = j.launches[i];
            if (!L.issued || L.dev != d) {
                li = std::min(li, i);
                continue;
            }
            if (L.dseq < p.head) continue;  // completed
            if (i < li) {
                li = i;
                block = (p.claim_open && L.dseq == p.claim_seq) ? p.claim_block : L.first_block;
            }
        }
        return DS_OK;
    }

    int wait_drained(Job& j, int timeout_ms) {
        const int d = j.dev;
        const int t = j.tenant[(size_t)d];
        const auto t0 = std::chrono::steady_clock::now();
        for (;;) {
            ds_progress p{};
            int st = ds_tenant_progress(dev(d).dom, t, &p);
            if (st) return st;
            if (p.drained || p.failed) return DS_OK;
            if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(timeout_ms))
                return ffail(DS_TIMEOUT, "job did not drain at a block boundary");
            std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
    }
};

extern "C" {

int ds_fleet_create(ds_fleet** out) {
    if (!out) return ffail(DS_INVALID_ARGUMENT, "null");
    *out = new ds_fleet();
    return DS_OK;
}

int ds_fleet_destroy(ds_fleet* f) {
    if (!f) return DS_OK;
    for (auto& j : f->jobs)
        for (auto& g : j.regions) {
            for (size_t d = 0; d < g.ptr.size(); ++d)
                if (g.owned[d] && g.ptr[d]) {
                    cudaSetDevice(f->devs[d].cuda);
                    cudaFree(g.ptr[d]);
                }
            if (g.lazy_ev) cudaEventDestroy(g.lazy_ev);
        }
    for (auto& d : f->devs) {
        cudaSetDevice(d.cuda);
        if (d.copy) cudaStreamDestroy(d.copy);
        if (d.lazy) cudaStreamDestroy(d.lazy);
    }
    delete f;
    return DS_OK;
}

int ds_fleet_add_device(ds_fleet* f, ds_domain* dom, int cuda_device, int standby, int* out) {
    if (!f || !dom || !out) return ffail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(f->mu);
    if (f->devs.size() >= 64) return ffail(DS_CONFIG_ERROR, "at most 64 devices");
    if (!f->jobs.empty()) return ffail(DS_CONFIG_ERROR, "add devices before jobs");
    ds_fleet::Device d;
    d.dom = dom;
    d.cuda = cuda_device;
    d.standby = standby != 0;
    if (cudaSetDevice(cuda_device) != cudaSuccess) return ffail(DS_NO_DEVICE, "bad device ordinal");
    cudaStreamCreateWithFlags(&d.copy, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&d.lazy, cudaStreamNonBlocking);
    f->devs.push_back(d);
    *out = (int)f->devs.size() - 1;
    return DS_OK;
}

int ds_fleet_add_job(ds_fleet* f, int dev, const ds_tenant_desc* desc, int* out) {
    if (!f || !desc || !out) return ffail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(f->mu);
    if (dev < 0 || dev >= (int)f->devs.size()) return ffail(DS_INVALID_ARGUMENT, "unknown device");
    if (f->devs[(size_t)dev].failed) return ffail(DS_CONFIG_ERROR, "device failed");
    ds_fleet::Job j;
    j.name = desc->name ? desc->name : "";
    j.priority = desc->priority;
    j.dev = dev;
    j.tenant.assign(f->devs.size(), -1);
    int st = f->ensure_tenant(j, dev);
    if (st) return st;
    f->jobs.push_back(std::move(j));
    *out = (int)f->jobs.size() - 1;
    return DS_OK;
}

int ds_fleet_add_region(ds_fleet* f, int job, void* ptr, uint64_t bytes, int* out) {
    if (!f || !ptr || !bytes || !out) return ffail(DS_INVALID_ARGUMENT, "null / empty region");
    std::lock_guard<std::mutex> g(f->mu);
    if (job < 0 || job >= (int)f->jobs.size()) return ffail(DS_INVALID_ARGUMENT, "unknown job");
    ds_fleet::Job& j = f->jobs[(size_t)job];
    if (!j.launches.empty()) return ffail(DS_CONFIG_ERROR, "regions are declared before launches");
    ds_fleet::Region r;
    r.bytes = bytes;
    r.ptr.assign(f->devs.size(), nullptr);
    r.owned.assign(f->devs.size(), false);
    r.ptr[(size_t)j.dev] = ptr;
    r.resident = 1ull << j.dev;  // the caller's buffer lives on the job's device
    j.regions.push_back(std::move(r));
    *out = (int)j.regions.size() - 1;
    return DS_OK;
}

int ds_fleet_add_kernel(ds_fleet* f, int job, const ds_kernel_desc* desc, const ds_reloc* relocs, int n_relocs,
                        const int32_t* touched, int n_touched, int* out) {
    if (!f || !desc || !out || n_relocs < 0 || n_touched < 0 || (n_relocs && !relocs) || (n_touched && !touched))
        return ffail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(f->mu);
    if (job < 0 || job >= (int)f->jobs.size()) return ffail(DS_INVALID_ARGUMENT, "unknown job");
    ds_fleet::Job& j = f->jobs[(size_t)job];
    ds_fleet::Kernel k;
    k.semantic_id = desc->semantic_id ? desc->semantic_id : "";
    k.desc = *desc;
    if (desc->args_size) k.args.assign((const uint8_t*)desc->args, (const uint8_t*)desc->args + desc->args_size);
    for (int i = 0; i < n_relocs; ++i) {
        if (relocs[i].region < 0 || relocs[i].region >= (int)j.regions.size())
            return ffail(DS_TRACE_VIOLATION, "relocation against a region outside the working set");
        if ((uint64_t)relocs[i].args_offset + 8 > k.args.size()) return ffail(DS_CONFIG_ERROR, "relocation past args");
        if (relocs[i].region_offset >= j.regions[(size_t)relocs[i].region].bytes)
            return ffail(DS_CONFIG_ERROR, "relocation offset past its region");
        k.relocs.push_back(relocs[i]);
    }
    for (int i = 0; i < n_touched; ++i) {
        // touched regions must lie in the working set (engine.cpp:176-181)
        if (touched[i] < 0 || touched[i] >= (int)j.regions.size())
            return ffail(DS_TRACE_VIOLATION, "kernel touches a region outside the working set");
        k.touched.push_back(touched[i]);
    }
    k.on_dev.assign(f->devs.size(), -1);
    j.kernels.push_back(std::move(k));
    const int id = (int)j.kernels.size() - 1;
    int st = f->register_on(j, id, j.dev);
    if (st) return st;
    *out = id;
    return DS_OK;
}

int ds_fleet_kernel_id(ds_fleet* f, int job, int kernel, int dev, int* out) {
    if (!f || !out) return ffail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(f->mu);
    if (job < 0 || job >= (int)f->jobs.size()) return ffail(DS_INVALID_ARGUMENT, "unknown job");
    ds_fleet::Job& j = f->jobs[(size_t)job];
    if (kernel < 0 || kernel >= (int)j.kernels.size() || dev < 0 || dev >= (int)f->devs.size())
        return ffail(DS_INVALID_ARGUMENT, "unknown kernel / device");
    *out = j.kernels[(size_t)kernel].on_dev[(size_t)dev];
    return DS_OK;
}

int ds_fleet_bind(ds_fleet* f, int job, int pctx) {
    if (!f) return ffail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(f->mu);
    if (job < 0 || job >= (int)f->jobs.size()) return ffail(DS_INVALID_ARGUMENT, "unknown job");
    ds_fleet::Job& j = f->jobs[(size_t)job];
    if (j.status) return ffail(DS_TENANT_FAILED, "job is not active");
    int st = ds_bind(f->dev(j.dev).dom, j.tenant[(size_t)j.dev], pctx);
    if (st) return st;
    j.pctx = pctx;
    return DS_OK;
}

int ds_fleet_launch(ds_fleet* f, int job, int kernel, uint64_t* fseq) {
    if (!f) return ffail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(f->mu);
    if (job < 0 || job >= (int)f->jobs.size()) return ffail(DS_INVALID_ARGUMENT, "unknown job");
    ds_fleet::Job& j = f->jobs[(size_t)job];
    if (kernel < 0 || kernel >= (int)j.kernels.size()) return ffail(DS_INVALID_ARGUMENT, "unknown kernel");
    // arrivals of a terminated vctx are dropped (engine.cpp:810-819)
    if (j.status) return ffail(DS_TENANT_FAILED, j.status == 2 ? "job stranded" : "job failed");
    ds_fleet::Launch L;
    L.kernel = kernel;
    j.launches.push_back(L);
    const size_t li = j.launches.size() - 1;
    int st = f->issue(j, li);
    if (st) {
        j.launches.pop_back();
        return st;
    }
    if (fseq) *fseq = li;
    return DS_OK;
}

int ds_fleet_wait(ds_fleet* f, int job, uint64_t fseq, int timeout_ms) {
    if (!f) return ffail(DS_INVALID_ARGUMENT, "null");
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        ds_domain* dom = nullptr;
        int tenant = -1;
        uint64_t dseq = 0;
        {
            std::lock_guard<std::mutex> g(f->mu);
            if (job < 0 || job >= (int)f->jobs.size()) return ffail(DS_INVALID_ARGUMENT, "unknown job");
            ds_fleet::Job& j = f->jobs[(size_t)job];
            if (fseq >= j.launches.size()) return ffail(DS_INVALID_ARGUMENT, "unknown launch");
            if (j.status) return ffail(DS_TENANT_FAILED, j.status == 2 ? "job stranded" : "job failed");
            const ds_fleet::Launch& L = j.launches[(size_t)fseq];
            dom = f->dev(L.dev).dom;
            tenant = j.tenant[(size_t)L.dev];
            dseq = L.dseq;
        }
        int st = ds_wait_tenant(dom, tenant, dseq, 20);
        if (st == DS_OK) {
            // the launch may have moved (global exception) while we waited
            std::lock_guard<std::mutex> g(f->mu);
            const ds_fleet::Launch& L = f->jobs[(size_t)job].launches[(size_t)fseq];
            if (f->dev(L.dev).dom == dom && L.dseq == dseq && !f->dev(L.dev).failed) return DS_OK;
            if (f->dev(L.dev).dom != dom || L.dseq != dseq) continue;
        }
        if (st != DS_OK && st != DS_TIMEOUT && st != DS_TENANT_FAILED) return st;
        if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(timeout_ms))
            return ffail(DS_TIMEOUT, "launch not complete");
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

int ds_fleet_migrate(ds_fleet* f, int job, int dst_dev, int dst_pctx, int timeout_ms) {
    if (!f) return ffail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(f->mu);
    if (job < 0 || job >= (int)f->jobs.size()) return ffail(DS_INVALID_ARGUMENT, "unknown job");
    if (dst_dev < 0 || dst_dev >= (int)f->devs.size()) return ffail(DS_INVALID_ARGUMENT, "unknown device");
    ds_fleet::Job& j = f->jobs[(size_t)job];
    if (j.status) return ffail(DS_TENANT_FAILED, "job is not active");
    if (f->dev(dst_dev).failed) return ffail(DS_CONFIG_ERROR, "destination failed");
    if (dst_dev == j.dev) {
        // same device: one control-word change, nothing to copy (shared address space)
        int st = ds_migrate(f->dev(dst_dev).dom, j.tenant[(size_t)dst_dev], dst_pctx);
        if (st) return st;
        j.pctx = dst_pctx;
        return DS_OK;
    }
    // a planned move happens between kernels (Remap at dispatch): the job's
    // issued launches finish on the source first
    const int src = j.dev;
    const int t = j.tenant[(size_t)src];
    for (const auto& L : j.launches) {
        if (!L.issued || L.dev != src) continue;
        int st = ds_wait_tenant(f->dev(src).dom, t, L.dseq, timeout_ms);
        if (st) return st;
    }
    if (j.pctx >= 0) ds_unbind(f->dev(src).dom, t);
    j.pctx = -1;
    return f->begin_migration(j, job, dst_dev, dst_pctx, false, j.launches.size(), 0);
}

int ds_fleet_global_exception(ds_fleet* f, int dv, int timeout_ms) {
    if (!f) return ffail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(f->mu);
    if (dv < 0 || dv >= (int)f->devs.size()) return ffail(DS_INVALID_ARGUMENT, "unknown device");
    ds_fleet::Device& D = f->dev(dv);
    if (D.failed) return DS_OK;
    D.failed = true;
    // the jobs on the device, in the order of its pctx pool (bound first,
    // engine.cpp:1102), then unbound ones by id
    int np = 0;
    ds_pctx_count(D.dom, &np);
    std::vector<int> order;
    std::vector<Frac_t> prior;
    for (int p = 0; p < np; ++p)
        for (size_t ji = 0; ji < f->jobs.size(); ++ji)
            if (f->jobs[ji].dev == dv && f->jobs[ji].status == 0 && f->jobs[ji].pctx == p) {
                order.push_back((int)ji);
                prior.push_back(f->tier_of(dv, p));
            }
    for (size_t ji = 0; ji < f->jobs.size(); ++ji)
        if (f->jobs[ji].dev == dv && f->jobs[ji].status == 0 && f->jobs[ji].pctx < 0) {
            order.push_back((int)ji);
            prior.push_back(Frac_t{0, 1});
        }
    // signal_preempt on every pctx of the device: the SMs leave at their next
    // logical-block boundary
    if (f->running(dv)) {
        std::vector<int32_t> none(DS_MAX_SMS, -1);
        int nsm = 0;
        ds_num_sms(D.dom, &nsm);
        int st = ds_quota_set(D.dom, none.data(), none.data(), nsm);
        if (st) return st;
        for (int ji : order) {
            ds_fleet::Job& j = f->jobs[(size_t)ji];
            if ((st = f->wait_drained(j, timeout_ms))) return st;
        }
    }
    std::vector<size_t> rli(order.size());
    std::vector<uint32_t> rblk(order.size());
    for (size_t i = 0; i < order.size(); ++i) {
        int st = f->resume_point(f->jobs[(size_t)order[i]], rli[i], rblk[i]);
        if (st) return st;
    }
    ds_stop(D.dom);  // the device is lost; its memory is read for the full eager copies
    for (size_t i = 0; i < order.size(); ++i) {
        ds_fleet::Job& j = f->jobs[(size_t)order[i]];
        j.pctx = -1;
        // emergency_migrate (engine.cpp:1124-1166): target on a standby device
        std::vector<int32_t> failed(f->devs.size()), standby(f->devs.size());
        std::vector<ds_place_pctx> pool;
        for (size_t d = 0; d < f->devs.size(); ++d) {
            failed[d] = f->devs[d].failed;
            standby[d] = f->devs[d].standby;
            if (f->devs[d].failed || !f->devs[d].standby) continue;
            int n = 0;
            ds_pctx_count(f->devs[d].dom, &n);
            for (int p = 0; p < n; ++p) {
                ds_place_pctx pp{};
                int nsm = 0, b = -1;
                ds_pctx_info(f->devs[d].dom, p, &pp.tier_num, &pp.tier_den, &nsm, &b);
                pp.device = (int32_t)d;
                pp.pctx = p;
                pp.bound = b >= 0;
                pool.push_back(pp);
            }
        }
        int target = -1;
        int st = ds_emergency_target(failed.data(), standby.data(), (int)f->devs.size(), pool.data(), (int)pool.size(),
                                     prior[i].num, prior[i].den, &target);
        if (st) return st;
        if (target < 0) {
            j.status = 2;  // Stranded (engine.cpp:1155-1160)
            f->ledger.stranded++;
            continue;
        }
        const int dst = pool[(size_t)target].device;
        f->dev(dst).standby = false;  // hosts live work from now on
        if ((st = f->begin_migration(j, order[i], dst, pool[(size_t)target].pctx, true, rli[i], rblk[i]))) return st;
    }
    return DS_OK;
}

int ds_fleet_job_get(ds_fleet* f, int job, ds_fleet_job_info* out) {
    if (!f || !out) return ffail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(f->mu);
    if (job < 0 || job >= (int)f->jobs.size()) return ffail(DS_INVALID_ARGUMENT, "unknown job");
    ds_fleet::Job& j = f->jobs[(size_t)job];
    f->advance_lazy(j);
    std::memset(out, 0, sizeof *out);
    out->device = j.dev;
    out->tenant = j.tenant[(size_t)j.dev];
    out->pctx = j.pctx;
    out->status = j.status;
    out->launches = j.launches.size();
    for (const auto& m : f->migrations) out->migrations += m.job == job;
    for (const auto& g2 : j.regions) out->lazy_pending += g2.lazy_dst >= 0;
    return DS_OK;
}

int ds_fleet_region(ds_fleet* f, int job, int region, int dev, void** ptr, int* resident, int* dirty) {
    if (!f) return ffail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(f->mu);
    if (job < 0 || job >= (int)f->jobs.size()) return ffail(DS_INVALID_ARGUMENT, "unknown job");
    ds_fleet::Job& j = f->jobs[(size_t)job];
    if (region < 0 || region >= (int)j.regions.size()) return ffail(DS_INVALID_ARGUMENT, "unknown region");
    f->advance_lazy(j);
    const ds_fleet::Region& r = j.regions[(size_t)region];
    if (dev < 0) dev = j.dev;
    if (dev >= (int)f->devs.size()) return ffail(DS_INVALID_ARGUMENT, "unknown device");
    if (ptr) *ptr = r.ptr[(size_t)dev];
    if (resident) *resident = (int)((r.resident >> dev) & 1ull);
    if (dirty) *dirty = r.dirty;
    return DS_OK;
}

int ds_fleet_read_region(ds_fleet* f, int job, int region, void* host, uint64_t bytes) {
    if (!f || !host) return ffail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(f->mu);
    if (job < 0 || job >= (int)f->jobs.size()) return ffail(DS_INVALID_ARGUMENT, "unknown job");
    ds_fleet::Job& j = f->jobs[(size_t)job];
    if (region < 0 || region >= (int)j.regions.size()) return ffail(DS_INVALID_ARGUMENT, "unknown region");
    f->advance_lazy(j);
    const ds_fleet::Region& r = j.regions[(size_t)region];
    if (bytes > r.bytes) return ffail(DS_INVALID_ARGUMENT, "read past the region");
    // the up-to-date copy: the job's device if resident there, else any other
    const int d = ((r.resident >> j.dev) & 1ull) ? j.dev : f->source_of(r, -1);
    if (d < 0) return ffail(DS_TRACE_VIOLATION, "region has no up-to-date copy");
    cudaSetDevice(f->dev(d).cuda);
    if (cudaMemcpyAsync(host, r.ptr[(size_t)d], bytes, cudaMemcpyDeviceToHost, f->dev(d).copy) != cudaSuccess ||
        cudaStreamSynchronize(f->dev(d).copy) != cudaSuccess)
        return ffail(DS_CUDA_ERROR, "region readback");
    return DS_OK;
}

int ds_fleet_migrations(ds_fleet* f, ds_migration_info* out, int cap, int* n) {
    if (!f || !n) return ffail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(f->mu);
    int k = 0;
    for (const auto& m : f->migrations) {
        if (out && k < cap) out[k] = m;
        ++k;
    }
    *n = k;
    return DS_OK;
}

int ds_fleet_ledger_get(ds_fleet* f, ds_fleet_ledger* out) {
    if (!f || !out) return ffail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(f->mu);
    *out = f->ledger;
    return DS_OK;
}

}  // extern "C"
