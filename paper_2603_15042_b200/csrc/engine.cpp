// GpuEngine — the reference SimEngine's dispatch loop (proj/src/engine/engine.cpp)
// driving the real executor instead of a performance model.
//
//   pump_launches  engine.cpp:1197-1248  -> pump()
//   apply_decision engine.cpp:688-754    -> apply()
//   start_or_resume engine.cpp:470-529   -> dispatch(): the record's kernels go
//                                           into the tenant's device ring once;
//                                           a paused record resumes in place
//   signal_preempt engine.cpp:756-806    -> ds_preempt(): SMs leave the victim
//                                           at their next logical-block boundary
//   begin_migration engine.cpp:620-672   -> ds_migrate(): one control-word change
//   finish_run     engine.cpp:830-906    -> finish(): transcript, predictor
//                                           (measured device duration), release
//
// One engine thread per domain polls device completions and runs the policy;
// API callers submit records (the reference's kernel arrivals).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/detshare/ds.h"
#include "policy.hpp"

using namespace detshare;

namespace {
thread_local std::string e_last_error;
int efail(int st, const std::string& w) {
    e_last_error = w;
    return st;
}
}  // namespace

struct ds_engine {
    struct Rec {
        LaunchRecord r;
        bool dispatched = false;
        bool done = false;
        uint64_t first_seq = 0, last_seq = 0;
        Time submit_host = 0, dispatch_host = 0, finish_host = 0;
        uint64_t t_first_claim = 0, t_end = 0;
        int pctx = -1;
        int preempted = 0;
        Time hang_needed = 0;  // arm_hang_check (engine.cpp:542-561): threshold x prediction
        bool hang_armed = false;
        bool failed = false;   // its job failed before it finished (never completes)
    };
    struct Job {
        int tenant = -1;
        PriorityClass prio = PriorityClass::BestEffort;
        std::deque<uint64_t> pending;  // not yet dispatched, program order
        int64_t running = -1;          // dispatched, unfinished record
        bool quarantined = false;
        int status = 0;                // VctxStatus: 0 Active, 1 Failed, 2 Stranded (types.hpp:77)
        Time last_finish = 0;
        bool has_last_finish = false;
        int64_t logical_progress = 0;
        std::vector<uint64_t> transcript;
        uint64_t fingerprint = 0;      // xor of its records' fingerprints at submit (engine.cpp:183-187)
    };

    ds_domain* dom = nullptr;
    PolicyConfig pcfg;
    std::unique_ptr<Policy> policy;
    DurationPredictor predictor;
    int release_on_idle = 1;
    int fair_handover = 1;
    int lend_tenant = -1;
    std::vector<Job> jobs;
    std::map<int, int> job_of_tenant;
    std::vector<Rec> recs;  // by id
    std::vector<int> pctx_bound;  // pctx -> job (-1)
    std::vector<Frac> pctx_tier;
    // a preempted pctx is unavailable while its SMs drain and the context
    // switches (on_preempt_boundary: unavailable for preempt_overhead,
    // engine.cpp:925-984); without it a best-effort victim rebinds the pctx in
    // the same pump and the launcher preempts it again, forever
    std::vector<Time> pctx_unavail_until;
    Time preempt_hold_ns = 200000;
    Time reset_delay_ns = 200000;  // EngineConfig.reset_delay (engine.hpp:65)
    std::mutex mu;
    std::thread th;
    std::atomic<bool> stop{false};
    std::atomic<bool> running{false};
    std::chrono::steady_clock::time_point t0;
    Time last_review = -1;
    Time next_review = -1;
    ds_engine_counters ctr{};
    // fault containment (engine.cpp:542-561, 1011-1035) and the JSONL event
    // log (engine.cpp:316-329, 1343-1352)
    bool hang_detection = false;
    double hang_threshold = 3.0;
    bool capture_log = false;
    uint64_t log_seq = 0;
    std::vector<std::string> event_log;
    struct Quarantine {
        int job;
        Frac tier;
        Time t;
    };
    std::vector<Quarantine> quarantines;
    ds_engine() : predictor(0.3, 1000000000) {}
    ds_ledger ledger0{};  // domain ledger at ds_engine_start

    // Kernel::fingerprint (types.cpp:39-48) of a launch record
    static uint64_t record_fingerprint(const LaunchRecord& r) {
        auto mix = [](uint64_t& h, uint64_t v) { h ^= v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2); };
        uint64_t h = 0x811c9dc5ULL;
        mix(h, r.signature.semantic_id.size());
        for (unsigned char c : r.signature.semantic_id) mix(h, c);
        mix(h, (uint64_t)r.signature.grid_size);
        mix(h, (uint64_t)r.base_duration);
        mix(h, (uint64_t)r.compute_saturation.num);
        mix(h, (uint64_t)r.compute_saturation.den);
        for (int32_t k : r.kernels) mix(h, (uint64_t)(uint32_t)k);
        return h;
    }

    // {"t","seq","kind",...} as the reference's log_event; t in engine ns
    void log(Time t, const char* kind, const std::string& fields) {
        if (!capture_log) return;
        std::string line = "{\"t\":\"" + std::to_string(t) + "\",\"seq\":" + std::to_string(log_seq++) +
                           ",\"kind\":\"" + kind + "\"";
        if (!fields.empty()) line += "," + fields;
        line += "}";
        event_log.push_back(std::move(line));
    }
    static std::string kv(const char* k, long long v) { return std::string("\"") + k + "\":" + std::to_string(v); }
    static std::string jstr(const std::string& v) {
        std::string o = "\"";
        for (char c : v) {
            if (c == '"' || c == '\\') o += '\\';
            o += c;
        }
        return o + "\"";
    }
    // KernelStart fields as the reference logs them (engine.cpp:519-525)
    std::string start_fields(int ji, const Rec& r, bool resumed) const {
        return kv("vctx", ji) + "," + kv("pctx", r.pctx) + ",\"kernel\":" + jstr(r.r.signature.semantic_id) + "," +
               kv("grid", r.r.signature.grid_size) + ",\"resumed\":" + (resumed ? "true" : "false");
    }

    Time now() const {
        return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    }
    int bound_pctx(int j) const {
        for (size_t p = 0; p < pctx_bound.size(); ++p)
            if (pctx_bound[p] == j) return (int)p;
        return -1;
    }
    const Rec* head(const Job& j) const {
        if (j.running >= 0) return &recs[j.running];
        if (j.pending.empty()) return nullptr;
        return &recs[j.pending.front()];
    }
    Time ready_time(const Job& j) const {
        if (j.running >= 0) return now();  // paused
        const Rec& r = recs[j.pending.front()];
        Time t = r.r.arrival;
        return t;
    }
    bool launchable(int ji) const {
        const Job& j = jobs[ji];
        if (j.running >= 0) return bound_pctx(ji) < 0;  // paused: needs a binding again
        if (j.pending.empty()) return false;
        return ready_time(j) <= now();
    }

    PolicyView build_view() const {
        PolicyView v;
        v.now = now();
        v.predictor = &predictor;
        Frac sum{0, 1}, mn{2, 1};
        for (size_t p = 0; p < pctx_tier.size(); ++p) {
            if (pctx_bound[p] >= 0) sum = sum + pctx_tier[p];
            if (pctx_tier[p] < mn) mn = pctx_tier[p];
        }
        v.bound_tier_sums[0] = sum;
        v.min_tiers[0] = mn;
        for (size_t p = 0; p < pctx_tier.size(); ++p) {
            PolicyView::PctxEntry e;
            e.id = (int)p;
            e.tier = pctx_tier[p];
            e.available = pctx_unavail_until[p] <= v.now;
            if (pctx_bound[p] >= 0) {
                e.bound = pctx_bound[p];
                const Job& j = jobs[pctx_bound[p]];
                if (j.running >= 0) {
                    const Rec& r = recs[j.running];
                    e.running_kernel = r.r.id;
                    e.running_signature = r.r.signature;
                    e.running_phase = r.r.phase;
                    e.running_priority = j.prio;
                    Time pred = predictor.predict(r.r.signature, r.r.base_duration);
                    Time el = v.now - r.dispatch_host;
                    e.running_remaining = pred > el ? pred - el : 0;
                }
            }
            v.pctxs.push_back(e);
        }
        for (size_t ji = 0; ji < jobs.size(); ++ji) {
            const Job& j = jobs[ji];
            PolicyView::VctxEntry e;
            e.id = (int)ji;
            e.priority = j.prio;
            e.quarantined = j.quarantined;
            e.bound = bound_pctx((int)ji) >= 0;
            e.pending = (int64_t)j.pending.size() + (j.running >= 0 ? 1 : 0);
            const Rec* h = head(j);
            if (h) e.head_phase = h->r.phase;
            e.decoding = h && h->r.phase == Phase::Decode;
            if (j.running >= 0 || !j.pending.empty()) v.active_vctx_count++;
            v.vctxs.push_back(e);
        }
        return v;
    }

    LaunchContext launch_context(int ji) const {
        LaunchContext lc;
        lc.vctx = ji;
        const Rec* h = head(jobs[ji]);
        if (h) {
            lc.kernel = &h->r;
            lc.slo = h->r.slo;
            lc.request_arrival = h->r.request_arrival;
        }
        return lc;
    }

    // apply_local_exception (engine.cpp:1049-1083): the job bound to the
    // faulting pctx fails — its records are dropped, it is unbound, and the
    // pctx is held unavailable for reset_delay.  The device already stopped
    // claiming its blocks (ds_fault_inject / a body's raise_fault), so the
    // other jobs keep running on their SMs untouched.
    void local_exception(int ji, uint32_t code) {
        Job& j = jobs[ji];
        if (j.status != 0) return;
        int p = bound_pctx(ji);
        Time t = now();
        log(t, "FaultInjected", std::string("\"fault\":\"local\",") + kv("pctx", p) + "," + kv("vctx", ji) + "," +
                                   kv("code", (long long)code));
        if (j.running >= 0) recs[j.running].failed = true;
        for (uint64_t id : j.pending) recs[id].failed = true;
        j.pending.clear();
        j.running = -1;
        j.status = 1;
        ctr.failed_jobs++;
        if (p >= 0) {
            ds_unbind(dom, j.tenant);
            pctx_bound[p] = -1;
            ctr.unbinds++;
            pctx_unavail_until[p] = t + reset_delay_ns;
            if (next_review < 0 || pctx_unavail_until[p] < next_review) next_review = pctx_unavail_until[p];
        }
    }
    void check_faults() {
        for (size_t ji = 0; ji < jobs.size(); ++ji) {
            if (jobs[ji].status != 0) continue;
            ds_fault_info f;
            if (ds_tenant_fault(dom, jobs[ji].tenant, &f) == DS_OK && f.code) local_exception((int)ji, f.code);
        }
    }

    // ---- mechanism ----
    int do_bind(int ji, int p) {
        int src = bound_pctx(ji);
        int rc = ds_migrate(dom, jobs[ji].tenant, p);
        if (rc) return rc;
        if (src >= 0) pctx_bound[src] = -1;
        pctx_bound[p] = ji;
        ctr.migrations++;
        log(now(), "MigrationDone", kv("vctx", ji) + "," + kv("pctx", p) + "," + kv("from", src));
        return 0;
    }
    void do_unbind(int ji) {
        int p = bound_pctx(ji);
        if (p < 0) return;
        ds_unbind(dom, jobs[ji].tenant);
        pctx_bound[p] = -1;
        ctr.unbinds++;
    }
    void dispatch(int ji) {
        Job& j = jobs[ji];
        if (j.running >= 0) {  // paused record resumes in place on its new binding
            Rec& pr = recs[j.running];
            pr.pctx = bound_pctx(ji);
            log(now(), "KernelStart", start_fields(ji, pr, true));
            return;
        }
        uint64_t id = j.pending.front();
        j.pending.pop_front();
        Rec& r = recs[id];
        for (size_t k = 0; k < r.r.kernels.size(); ++k) {
            uint64_t seq = 0;
            ds_launch(dom, j.tenant, r.r.kernels[k], id, &seq);
            if (k == 0) r.first_seq = seq;
            r.last_seq = seq;
        }
        r.dispatched = true;
        r.dispatch_host = now();
        r.pctx = bound_pctx(ji);
        j.running = (int64_t)id;
        ctr.dispatches++;
        if (hang_detection && !j.quarantined) {
            r.hang_needed = (Time)(hang_threshold * (double)predictor.predict(r.r.signature, r.r.base_duration));
            r.hang_armed = true;
        }
        log(r.dispatch_host, "KernelStart", start_fields(ji, r, false));
    }

    enum Outcome { kDirect, kRemap, kDeferPolicy, kDeferError };
    Outcome apply(int ji, const PolicyDecision& d) {
        using K = PolicyDecision::Kind;
        auto fail = [&]() {
            ctr.policy_errors++;
            return kDeferError;
        };
        switch (d.kind) {
            case K::NoAction:
            case K::DispatchDefer: return kDeferPolicy;
            case K::DispatchDirect: {
                int p = bound_pctx(ji);
                if (p < 0) return fail();                               // direct dispatch while unbound
                if (pctx_unavail_until[p] > now()) return fail();       // pctx not available
                if (jobs[ji].running >= 0 && recs[jobs[ji].running].dispatched && p >= 0 && !launchable(ji))
                    return fail();
                dispatch(ji);
                return kDirect;
            }
            case K::DispatchRemap: {
                if (d.target < 0 || d.target >= (int)pctx_tier.size()) return fail();
                if (pctx_bound[d.target] >= 0) return fail();
                if (pctx_unavail_until[d.target] > now()) return fail();
                Frac sum{0, 1};
                for (size_t p = 0; p < pctx_tier.size(); ++p)
                    if (pctx_bound[p] >= 0) sum = sum + pctx_tier[p];
                if (sum + pctx_tier[d.target] > Frac{1, 1}) return fail();  // spatial feasibility
                if (jobs[ji].quarantined) {  // quarantined vctx above minimal tier (engine.cpp:726-728)
                    Frac mn{2, 1};
                    for (const auto& f : pctx_tier)
                        if (f < mn) mn = f;
                    if (pctx_tier[d.target] != mn) return fail();
                }
                if (do_bind(ji, d.target)) return fail();
                dispatch(ji);
                return kRemap;
            }
            case K::Preempt: {
                if (d.target < 0 || d.target >= (int)pctx_tier.size()) return fail();
                int victim = pctx_bound[d.target];
                if (victim < 0) return kDeferPolicy;  // no-op (engine.cpp:738-746)
                if (victim == ji) return fail();      // self-preemption
                ds_preempt(dom, d.target);
                pctx_bound[d.target] = -1;
                hold(d.target);
                log(now(), "PreemptSignal", kv("vctx", victim) + "," + kv("pctx", d.target) + "," + kv("by", ji));
                if (jobs[victim].running >= 0) recs[jobs[victim].running].preempted++;
                ctr.preemptions++;
                return kDeferPolicy;
            }
        }
        return kDeferPolicy;
    }

    void hold(int p) {
        pctx_unavail_until[p] = now() + preempt_hold_ns;
        if (next_review < 0 || pctx_unavail_until[p] < next_review) next_review = pctx_unavail_until[p];
    }

    bool pool_exhausted() const {
        Frac sum{0, 1};
        for (size_t p = 0; p < pctx_tier.size(); ++p)
            if (pctx_bound[p] >= 0) sum = sum + pctx_tier[p];
        for (size_t p = 0; p < pctx_tier.size(); ++p)
            if (pctx_bound[p] < 0 && sum + pctx_tier[p] <= Frac{1, 1}) return false;
        return true;
    }

    void temporal_handover() {
        auto* tp = dynamic_cast<TemporalBaselinePolicy*>(policy.get());
        if (!tp || !fair_handover) return;
        PolicyView v = build_view();
        auto owner = tp->owner_at(v);
        if (!owner) return;
        for (size_t p = 0; p < pctx_bound.size(); ++p) {
            int holder = pctx_bound[p];
            if (holder >= 0 && holder != *owner && launchable_or_pending(*owner)) {
                ds_preempt(dom, (int)p);
                pctx_bound[p] = -1;
                hold((int)p);
                if (jobs[holder].running >= 0) recs[jobs[holder].running].preempted++;
                ctr.preemptions++;
            }
        }
    }
    bool launchable_or_pending(int ji) const { return jobs[ji].running >= 0 || !jobs[ji].pending.empty(); }

    void pump() {
        temporal_handover();
        bool changed = true;
        int guard = 0;
        while (changed && ++guard < 10000) {
            changed = false;
            std::vector<int> ready;
            for (size_t ji = 0; ji < jobs.size(); ++ji)
                if (launchable((int)ji)) ready.push_back((int)ji);
            if (ready.empty()) break;
            std::stable_sort(ready.begin(), ready.end(), [&](int a, int b) {
                int ka = policy->launch_order_key(launch_context(a));
                int kb = policy->launch_order_key(launch_context(b));
                if (ka != kb) return ka < kb;
                if (jobs[a].prio != jobs[b].prio) return jobs[a].prio == PriorityClass::LatencyCritical;
                return a < b;
            });
            for (int ji : ready) {
                if (!launchable(ji)) continue;
                PolicyView view = build_view();
                LaunchContext lc = launch_context(ji);
                ctr.decisions++;
                Outcome o = apply(ji, policy->on_launch(view, lc));
                if (o == kDirect || o == kRemap) {
                    changed = true;
                    continue;
                }
                bool unbound = bound_pctx(ji) < 0;
                if (unbound && o == kDeferPolicy && pool_exhausted()) {
                    lc.pool_exhausted = true;
                    PolicyView v2 = build_view();
                    PolicyDecision d2 = policy->on_congestion(v2, lc);
                    if (d2.kind == PolicyDecision::Kind::Preempt) {
                        apply(ji, d2);
                        changed = true;  // capacity freed now (SMs yield at block boundaries)
                    }
                }
            }
        }
        // review tick for time-driven policies (engine.cpp:1250-1265)
        bool waiting = false;
        for (size_t ji = 0; ji < jobs.size(); ++ji) waiting |= launchable((int)ji) || jobs[ji].running >= 0;
        if (waiting) {
            auto t = policy->next_review_time(build_view());
            if (t && *t > now()) next_review = *t;
        }
    }

    void finish(int ji, Rec& r) {
        Job& j = jobs[ji];
        r.done = true;
        r.finish_host = now();
        j.running = -1;
        j.transcript.push_back(r.r.id);
        j.logical_progress++;
        j.last_finish = r.finish_host;
        j.has_last_finish = true;
        if (r.t_end > r.t_first_claim) predictor.observe(r.r.signature, (Time)(r.t_end - r.t_first_claim));
        ctr.completed++;
        // engine.cpp:871-877: exec = the run's executed time (device ns here)
        log(r.finish_host, "KernelFinish",
            kv("vctx", ji) + "," + kv("pctx", r.pctx) + ",\"kernel\":" + jstr(r.r.signature.semantic_id) + "," +
                kv("grid", r.r.signature.grid_size) + ",\"exec\":\"" +
                std::to_string((long long)(r.t_end - r.t_first_claim)) + "\"");
        {
            PolicyView v = build_view();
            PolicyDecision d = policy->on_completion(v, launch_context(ji));
            if (d.kind == PolicyDecision::Kind::Preempt) apply(ji, d);
        }
        if (release_on_idle) {
            bool next_ready = !j.pending.empty() && recs[j.pending.front()].r.arrival <= now();
            if (!next_ready) do_unbind(ji);
        }
    }

    // on_hang_check (engine.cpp:1011-1035): a record running longer than
    // threshold x its prediction marks its vctx quarantined — its SMs yield at
    // the next logical-block boundary and it may only bind the pool's minimum
    // tier from then on (eligible_bind) — so a soft-hung tenant is confined to
    // the smallest SM set instead of holding its quota
    void hang_check(Time t) {
        for (size_t ji = 0; ji < jobs.size(); ++ji) {
            Job& j = jobs[ji];
            if (j.quarantined || j.running < 0) continue;
            Rec& r = recs[j.running];
            if (!r.hang_armed || t - r.dispatch_host < r.hang_needed) continue;
            Frac mn{2, 1};
            for (const auto& f : pctx_tier)
                if (f < mn) mn = f;
            j.quarantined = true;
            quarantines.push_back({(int)ji, mn, t});
            log(t, "HangCheck", kv("vctx", (long long)ji) + "," + kv("pctx", bound_pctx((int)ji)) +
                                    ",\"flagged\":true," + kv("elapsed", t - r.dispatch_host));
            int p = bound_pctx((int)ji);
            if (p >= 0 && pctx_tier[p] != mn) {
                ds_preempt(dom, p);
                pctx_bound[p] = -1;
                hold(p);
                r.preempted++;
                ctr.preemptions++;
            }
        }
    }

    void loop() {
        std::vector<ds_completion> buf(4096);
        auto last_active = std::chrono::steady_clock::now();
        while (!stop.load()) {
            bool work = false;
            {
                std::lock_guard<std::mutex> g(mu);
                int n = 0;
                ds_poll(dom, buf.data(), (int)buf.size(), &n);
                for (int i = 0; i < n; ++i) {
                    const ds_completion& c = buf[i];
                    auto it = job_of_tenant.find(c.tenant);
                    if (it == job_of_tenant.end()) continue;
                    Job& j = jobs[it->second];
                    if (j.running < 0) continue;
                    Rec& r = recs[j.running];
                    if (c.seq == r.first_seq) r.t_first_claim = c.t_first_claim;
                    if (c.seq == r.last_seq) {
                        r.t_end = c.t_end;
                        finish(it->second, r);
                    }
                    work = true;
                }
                check_faults();
                Time t = now();
                if (hang_detection) hang_check(t);
                bool review = next_review >= 0 && t >= next_review;
                if (review) next_review = -1;
                bool arrivals = false;
                for (size_t ji = 0; ji < jobs.size(); ++ji) arrivals |= launchable((int)ji);
                if (work || review || arrivals) pump();
            }
            // busy-poll (pause) while work is recent: a sleep costs the timer
            // slack (~50 us) on every decode step's completion -> next launch
            if (work) {
                last_active = std::chrono::steady_clock::now();
            } else if (std::chrono::steady_clock::now() - last_active < std::chrono::milliseconds(20)) {
#if defined(__x86_64__) || defined(__i386__)
                for (int i = 0; i < 32; ++i) __builtin_ia32_pause();
#endif
            } else {
                std::this_thread::sleep_for(std::chrono::microseconds(5));
            }
        }
    }
};

extern "C" {

const char* ds_engine_last_error(void) { return e_last_error.c_str(); }

static int engine_create(ds_domain* dom, const ds_engine_config* cfg, const ds_policy_vtable* vt, void* user,
                         ds_engine** out) {
    if (!dom || !cfg || !out) return efail(DS_INVALID_ARGUMENT, "null");
    if (vt && !vt->on_launch) return efail(DS_CONFIG_ERROR, "a policy needs on_launch");
    auto* e = new ds_engine();
    e->dom = dom;
    e->pcfg.name = vt ? (vt->name ? vt->name : "user") : (cfg->policy ? cfg->policy : "slo-aware");
    if (cfg->quantum_ns > 0) e->pcfg.quantum = cfg->quantum_ns;
    if (cfg->alpha > 0) e->pcfg.predictor_alpha = cfg->alpha;
    if (cfg->cold_start_ns > 0) e->pcfg.cold_start_prediction = cfg->cold_start_ns;
    for (int i = 0; i < cfg->n_assignments && i < 64; ++i) e->pcfg.assignments[cfg->assign_vctx[i]] = cfg->assign_pctx[i];
    try {
        // SimEngine(Scenario, std::unique_ptr<Policy>) (engine.hpp:155): a
        // user policy replaces the named one
        e->policy = vt ? make_abi_policy(*vt, user) : make_policy(e->pcfg);
        e->predictor = DurationPredictor(e->pcfg.predictor_alpha, e->pcfg.cold_start_prediction);
    } catch (const std::exception& ex) {
        delete e;
        return efail(DS_CONFIG_ERROR, ex.what());
    }
    e->release_on_idle = cfg->release_on_idle;
    e->hang_detection = cfg->hang_detection != 0;
    if (cfg->hang_threshold > 0) e->hang_threshold = cfg->hang_threshold;
    e->capture_log = cfg->capture_log != 0;
    if (cfg->reset_delay_ns > 0) e->reset_delay_ns = cfg->reset_delay_ns;
    e->fair_handover = cfg->fair_handover;
    e->lend_tenant = cfg->lend_tenant;
    int np = 0;
    ds_pctx_count(dom, &np);
    bool has_full = false;
    for (int p = 0; p < np; ++p) {
        int64_t num = 0, den = 1;
        int nsm = 0, bound = -1;
        ds_pctx_info(dom, p, &num, &den, &nsm, &bound);
        e->pctx_tier.push_back(Frac{num, den});
        e->pctx_bound.push_back(-1);
        e->pctx_unavail_until.push_back(0);
        if (num == den) has_full = true;
    }
    if (!vt && e->pcfg.name == "temporal" && !has_full) {  // engine.cpp:193-202
        delete e;
        return efail(DS_CONFIG_ERROR, "temporal baseline needs a full-tier pctx in the pool");
    }
    *out = e;
    return DS_OK;
}

int ds_engine_create(ds_domain* dom, const ds_engine_config* cfg, ds_engine** out) {
    return engine_create(dom, cfg, nullptr, nullptr, out);
}

int ds_engine_create_with_policy(ds_domain* dom, const ds_engine_config* cfg, const ds_policy_vtable* vt, void* user,
                                 ds_engine** out) {
    if (!vt) return efail(DS_INVALID_ARGUMENT, "null policy vtable");
    return engine_create(dom, cfg, vt, user, out);
}

int ds_engine_snapshot(ds_engine* e, ds_view* out) {
    if (!e || !out) return efail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(e->mu);
    PolicyView v = e->build_view();
    view_to_c(v, out);
    out->predictor = nullptr;  // the snapshot outlives the lock: no live pointers
    for (int i = 0; i < out->n_pctx; ++i) out->pctx[i].running_semantic_id = nullptr;
    return DS_OK;
}

int ds_engine_destroy(ds_engine* e) {
    if (!e) return DS_OK;
    ds_engine_stop(e);
    delete e;
    return DS_OK;
}

int ds_engine_add_job(ds_engine* e, int tenant, int priority, int* job) {
    if (!e || !job) return efail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(e->mu);
    ds_engine::Job j;
    j.tenant = tenant;
    j.prio = priority == DS_LATENCY_CRITICAL ? PriorityClass::LatencyCritical : PriorityClass::BestEffort;
    e->jobs.push_back(j);
    *job = (int)e->jobs.size() - 1;
    e->job_of_tenant[tenant] = *job;
    return DS_OK;
}

int ds_engine_submit(ds_engine* e, int job, const ds_record_desc* d, uint64_t* rec_id) {
    if (!e || !d || !rec_id) return efail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(e->mu);
    if (job < 0 || job >= (int)e->jobs.size()) return efail(DS_INVALID_ARGUMENT, "unknown job");
    if (d->n_kernels < 1 || !d->kernels) return efail(DS_CONFIG_ERROR, "record needs >= 1 kernel");
    if (d->sat_den <= 0 || d->sat_num <= 0 || d->sat_num > d->sat_den)
        return efail(DS_CONFIG_ERROR, "compute_saturation must lie in (0, 1]");  // engine.cpp:163-165
    ds_engine::Rec r;
    r.r.id = e->recs.size();
    r.r.job = job;
    r.r.signature.semantic_id = d->semantic_id ? d->semantic_id : "";
    r.r.signature.grid_size = d->grid_size;
    r.r.base_duration = d->base_hint_ns > 0 ? d->base_hint_ns : 0;
    r.r.compute_saturation = Frac{d->sat_num, d->sat_den};
    r.r.phase = (Phase)d->phase;
    r.r.request = d->request;
    r.r.decode_index = d->decode_index;
    if (d->tpot_ns > 0 || d->ttft_ns > 0) r.r.slo = SloSpec{d->ttft_ns, d->tpot_ns};
    Time now = e->running ? e->now() : 0;
    r.r.arrival = d->arrival_ns > 0 ? d->arrival_ns : now;
    r.r.request_arrival = d->request_arrival_ns > 0 ? d->request_arrival_ns : r.r.arrival;
    r.r.kernels.assign(d->kernels, d->kernels + d->n_kernels);
    r.submit_host = now;
    // arrival floors are non-decreasing per job (engine.cpp:172-176)
    auto& jb = e->jobs[job];
    // arrivals of a failed vctx are dropped (engine.cpp:810-819)
    if (jb.status != 0) return efail(DS_TENANT_FAILED, "job failed (local exception)");
    if (!jb.pending.empty() && e->recs[jb.pending.back()].r.arrival > r.r.arrival)
        return efail(DS_CONFIG_ERROR, "kernel arrival floors must be non-decreasing");
    jb.fingerprint ^= ds_engine::record_fingerprint(r.r);
    e->recs.push_back(std::move(r));
    jb.pending.push_back(e->recs.back().r.id);
    *rec_id = e->recs.back().r.id;
    e->log(now, "Arrival", ds_engine::kv("vctx", job) + "," + ds_engine::kv("kernel_id", (long long)*rec_id));
    return DS_OK;
}

int ds_engine_start(ds_engine* e) {
    if (!e) return efail(DS_INVALID_ARGUMENT, "null");
    if (e->running) return efail(DS_ALREADY_RUNNING, "engine running");
    if (e->lend_tenant >= 0) ds_set_lend(e->dom, e->lend_tenant);
    ds_ledger_get(e->dom, &e->ledger0);
    e->t0 = std::chrono::steady_clock::now();
    e->stop = false;
    e->running = true;
    e->th = std::thread([e] { e->loop(); });
    return DS_OK;
}

int ds_engine_stop(ds_engine* e) {
    if (!e) return efail(DS_INVALID_ARGUMENT, "null");
    if (!e->running) return DS_OK;
    e->stop = true;
    e->th.join();
    e->running = false;
    // finalize (engine.cpp:1370-1383): kernel records must be unchanged — the
    // engine's launch records and the device kernels' argument blocks
    std::vector<uint64_t> fp(e->jobs.size(), 0);
    for (const auto& r : e->recs) fp[r.r.job] ^= ds_engine::record_fingerprint(r.r);
    for (size_t j = 0; j < e->jobs.size(); ++j)
        if (fp[j] != e->jobs[j].fingerprint)
            return efail(DS_RECORD_MUTATED, "launch records of job " + std::to_string(j) + " mutated during the run");
    int bad = -1;
    if (ds_verify_kernels(e->dom, &bad) == DS_RECORD_MUTATED)
        return efail(DS_RECORD_MUTATED, std::string("kernel records mutated during the run: ") + ds_last_error());
    return DS_OK;
}

int ds_engine_ledger(ds_engine* e, ds_ledger* out) {
    if (!e || !out) return efail(DS_INVALID_ARGUMENT, "null");
    ds_ledger now{};
    int rc = ds_ledger_get(e->dom, &now);
    if (rc) return efail(rc, ds_last_error());
    out->ctx_switches = now.ctx_switches - e->ledger0.ctx_switches;
    out->ctx_switch_total_ns = now.ctx_switch_total_ns - e->ledger0.ctx_switch_total_ns;
    out->preemptions = now.preemptions - e->ledger0.preemptions;
    out->preempt_total_ns = now.preempt_total_ns - e->ledger0.preempt_total_ns;
    out->migrations = now.migrations - e->ledger0.migrations;
    out->migration_total_ns = now.migration_total_ns - e->ledger0.migration_total_ns;
    out->demand_faults = 0;
    out->demand_fault_total_ns = 0;
    return DS_OK;
}

int ds_engine_job_fingerprint(ds_engine* e, int job, uint64_t* fp) {
    if (!e || !fp) return efail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(e->mu);
    if (job < 0 || job >= (int)e->jobs.size()) return efail(DS_INVALID_ARGUMENT, "unknown job");
    *fp = e->jobs[job].fingerprint;
    return DS_OK;
}

int ds_engine_now(ds_engine* e, int64_t* ns) {
    if (!e || !ns) return efail(DS_INVALID_ARGUMENT, "null");
    *ns = e->running ? e->now() : 0;
    return DS_OK;
}

int ds_engine_wait(ds_engine* e, uint64_t rec_id, int timeout_ms) {
    if (!e) return efail(DS_INVALID_ARGUMENT, "null");
    auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms < 0 ? 1 << 30 : timeout_ms);
    for (;;) {
        {
            std::lock_guard<std::mutex> g(e->mu);
            if (rec_id >= e->recs.size()) return efail(DS_INVALID_ARGUMENT, "unknown record");
            if (e->recs[rec_id].done) return DS_OK;
            if (e->recs[rec_id].failed) return efail(DS_TENANT_FAILED, "record's job failed (local exception)");
        }
        if (std::chrono::steady_clock::now() > deadline) return efail(DS_TIMEOUT, "record wait timed out");
        std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

int ds_engine_record(ds_engine* e, uint64_t rec_id, ds_record_info* out) {
    if (!e || !out) return efail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(e->mu);
    if (rec_id >= e->recs.size()) return efail(DS_INVALID_ARGUMENT, "unknown record");
    const auto& r = e->recs[rec_id];
    out->id = r.r.id;
    out->job = r.r.job;
    out->state = r.done ? 2 : (r.failed ? 3 : (r.dispatched ? 1 : 0));
    out->pctx = r.pctx;
    out->preempted = r.preempted;
    out->phase = (int)r.r.phase;
    out->request = r.r.request;
    out->decode_index = r.r.decode_index;
    out->arrival_host_ns = r.r.arrival;
    out->dispatch_host_ns = r.dispatch_host;
    out->finish_host_ns = r.finish_host;
    out->t_first_claim = r.t_first_claim;
    out->t_end = r.t_end;
    out->first_seq = r.first_seq;
    out->last_seq = r.last_seq;
    return DS_OK;
}

int ds_engine_counters_get(ds_engine* e, ds_engine_counters* out) {
    if (!e || !out) return efail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(e->mu);
    *out = e->ctr;
    return DS_OK;
}

int ds_engine_transcript(ds_engine* e, int job, uint64_t* rec_ids, int cap, int* n) {
    if (!e || !n) return efail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(e->mu);
    if (job < 0 || job >= (int)e->jobs.size()) return efail(DS_INVALID_ARGUMENT, "unknown job");
    const auto& t = e->jobs[job].transcript;
    int m = std::min<int>(cap, (int)t.size());
    for (int i = 0; i < m; ++i) rec_ids[i] = t[i];
    *n = (int)t.size();
    return DS_OK;
}

int ds_engine_predict(ds_engine* e, const char* semantic_id, int64_t grid, int64_t* ns) {
    if (!e || !ns) return efail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(e->mu);
    *ns = e->predictor.predict(KernelSignature{semantic_id ? semantic_id : "", grid});
    return DS_OK;
}

int ds_engine_event_log(ds_engine* e, char* out, int64_t cap, int64_t* len) {
    if (!e || !len) return efail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(e->mu);
    std::string s;
    for (const auto& l : e->event_log) s += l + "\n";
    *len = (int64_t)s.size();
    if (out && cap > 0) {
        int64_t m = std::min<int64_t>(cap - 1, (int64_t)s.size());
        std::memcpy(out, s.data(), (size_t)m);
        out[m] = 0;
    }
    return DS_OK;
}

int ds_engine_quarantines(ds_engine* e, int32_t* jobs, int64_t* t_ns, int cap, int* n) {
    if (!e || !n) return efail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(e->mu);
    int m = std::min<int>(cap, (int)e->quarantines.size());
    for (int i = 0; i < m; ++i) {
        if (jobs) jobs[i] = e->quarantines[i].job;
        if (t_ns) t_ns[i] = e->quarantines[i].t;
    }
    *n = (int)e->quarantines.size();
    return DS_OK;
}

int ds_engine_fault_local(ds_engine* e, int pctx) {
    if (!e) return efail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(e->mu);
    if (pctx < 0 || pctx >= (int)e->pctx_bound.size()) return efail(DS_INVALID_ARGUMENT, "unknown pctx");
    const int ji = e->pctx_bound[pctx];
    if (ji < 0) {  // engine.cpp:1051-1058: no bound vctx, no effect
        e->log(e->now(), "FaultInjected", std::string("\"fault\":\"local\",") + ds_engine::kv("pctx", pctx) +
                                              ",\"effect\":\"none\"");
        return DS_OK;
    }
    int rc = ds_fault_inject(e->dom, e->jobs[ji].tenant, DS_FAULT_INJECTED);
    if (rc) return efail(rc, "fault injection");
    e->local_exception(ji, DS_FAULT_INJECTED);
    return DS_OK;
}

int ds_engine_job_status(ds_engine* e, int job, int* status) {
    if (!e || !status) return efail(DS_INVALID_ARGUMENT, "null");
    std::lock_guard<std::mutex> g(e->mu);
    if (job < 0 || job >= (int)e->jobs.size()) return efail(DS_INVALID_ARGUMENT, "unknown job");
    *status = e->jobs[job].status;
    return DS_OK;
}

int ds_policy_names(char* out, int cap) {
    std::string s;
    for (const auto& n : policy_names()) s += (s.empty() ? "" : ",") + n;
    if (!out || (int)s.size() + 1 > cap) return efail(DS_INVALID_ARGUMENT, "buffer");
    std::memcpy(out, s.c_str(), s.size() + 1);
    return DS_OK;
}

}  // extern "C"
