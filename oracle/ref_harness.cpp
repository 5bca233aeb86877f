// ORACLE HARNESS — test infrastructure only.
//
// extern "C" entry points over the reference library (corosim, compiled
// unmodified from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libcorosim_ref.so).  Used by tests/test_oracle_ref.py to pin the
// restatements (oracle/numlab.py, oracle/cnumlab.c) and by bench.py's
// reference arm / cpu_baseline leg to time the reference simulator.
#include "corosim/engine/engine.hpp"
#include "corosim/io/metrics.hpp"
#include "corosim/io/scenario.hpp"
#include "corosim/io/trace.hpp"
#include "corosim/io/workload.hpp"
#include "corosim/numlab/equivalence.hpp"
#include "corosim/numlab/float_format.hpp"
#include "corosim/numlab/reduction.hpp"
#include "corosim/policy/policies.hpp"
#include "corosim/runtime/migration.hpp"
#include "corosim/rational.hpp"

#include <json.hpp>

#include "policy_case.h"

#include <algorithm>
#include <chrono>
#include <csetjmp>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <cstring>
#include <sstream>
#include <string>

using namespace corosim;

// The reference checks its invariants with assert(); an assertion inside the
// simulator must not abort the process that hosts the checker, so the harness
// supplies glibc's assertion handler (bound locally, -Bsymbolic) and longjmps
// back to the entry point, which reports the failed check as an error string
// (glibc declares the handler noexcept, so it cannot throw).  No reference
// source is changed; the same check still fires.  The abandoned simulation's
// memory is leaked — acceptable on this error path.
namespace {
thread_local std::jmp_buf* g_assert_jmp = nullptr;
thread_local std::string g_assert_msg;
}  // namespace

extern "C" void __assert_fail(const char* expr, const char* file, unsigned int line, const char* func) {
    g_assert_msg = std::string("reference assertion failed: ") + expr + " (" + file + ":" + std::to_string(line) +
                   ", " + func + ")";
    if (g_assert_jmp) std::longjmp(*g_assert_jmp, 1);
    std::fprintf(stderr, "%s\n", g_assert_msg.c_str());
    std::abort();
}

#define REF_GUARDED(out, cap, body)                       \
    do {                                                  \
        std::jmp_buf jb;                                  \
        if (setjmp(jb)) {                                 \
            g_assert_jmp = nullptr;                       \
            put(std::string("error: ") + g_assert_msg, out, cap); \
            return 2;                                     \
        }                                                 \
        g_assert_jmp = &jb;                               \
        int rc_ = [&]() -> int { body }();                \
        g_assert_jmp = nullptr;                           \
        return rc_;                                       \
    } while (0)

namespace {

std::string fv_str(const FloatValue& v) {
    switch (v.cls) {
        case FloatValue::Cls::Finite:
            return numerator(v.value).str() + "/" + denominator(v.value).str();
        case FloatValue::Cls::PosInf: return "inf";
        case FloatValue::Cls::NegInf: return "-inf";
        case FloatValue::Cls::NaN: return "nan";
    }
    return "?";
}

int put(const std::string& s, char* out, long cap) {
    if (!out || cap <= 0) return -1;
    if (static_cast<long>(s.size()) + 1 > cap) return -2;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
}

FloatFormatKind kind_of(int fmt) {
    return fmt == 0 ? FloatFormatKind::FP16 : fmt == 1 ? FloatFormatKind::BF16 : FloatFormatKind::FP32;
}

}  // namespace

// migrations (migration.hpp:34-45), vctx status, ledger and the event log:
// the emergency-migration / working-set parity tests read them
static void add_migrations(nlohmann::ordered_json& j, const SimulationReport& rep) {
    nlohmann::ordered_json mig = nlohmann::ordered_json::array();
    for (const auto& m : rep.migrations) {
        mig.push_back({{"vctx", m.vctx.value},
                       {"src", m.src.valid() ? m.src.value : -1},
                       {"dst", m.dst.value},
                       {"eager_bytes", m.eager_bytes},
                       {"lazy_bytes", m.lazy_bytes},
                       {"start", to_decimal_string(m.start)},
                       {"end", to_decimal_string(m.end)},
                       {"demand_faults", m.demand_faults},
                       {"emergency", m.emergency},
                       {"aborted", m.aborted}});
    }
    j["migrations"] = mig;
    nlohmann::ordered_json vs;
    for (const auto& [vid, stt] : rep.vctx_status) vs[std::to_string(vid.value)] = static_cast<int>(stt);
    j["vctx_status"] = vs;
    j["ledger"] = {{"migrations", rep.ledger.migrations},
                   {"demand_faults", rep.ledger.demand_faults},
                   {"migration_total", to_decimal_string(rep.ledger.migration_total)},
                   {"demand_fault_total", to_decimal_string(rep.ledger.demand_fault_total)}};
    j["event_log"] = rep.event_log;
}

extern "C" {

// reduction_result (equivalence.cpp:19-25) as "num/den" | "inf" | "-inf" | "nan"
int ref_reduction_result(unsigned long long seed, long long n, int fmt, long long grid, char* out,
                         long cap) {
    try {
        ReductionSpec spec{n, seed, kind_of(fmt)};
        return put(fv_str(reduction_result(spec, grid)), out, cap);
    } catch (const std::exception& e) {
        put(std::string("error: ") + e.what(), out, cap);
        return 1;
    }
}

// seeded_values (equivalence.cpp:7-17): value i as "num/den"
int ref_seeded_value(unsigned long long seed, long long n, int fmt, long long i, char* out, long cap) {
    auto v = seeded_values(seed, n, kind_of(fmt));
    if (i < 0 || i >= n) return 1;
    return put(fv_str(v[static_cast<std::size_t>(i)]), out, cap);
}

// round_to (float_format.cpp:43-67) on an exact rational num/den
int ref_round_to(int fmt, const char* num, const char* den, char* out, long cap) {
    try {
        BigInt bn{std::string(num)};
        BigInt bd{std::string(den)};
        Rational r(bn, bd);
        return put(fv_str(round_to(FloatFormat::of(kind_of(fmt)), r)), out, cap);
    } catch (const std::exception& e) {
        put(std::string("error: ") + e.what(), out, cap);
        return 1;
    }
}

// reduce_with_plan over explicit values given as exact decimal lines with
// balanced(n, g) bounds; tree != 0 selects combine_tree.
int ref_reduce_values(int fmt, const char* values_nl, long long n, long long g, int tree, char* out,
                      long cap) {
    try {
        std::vector<FloatValue> vals;
        const char* p = values_nl;
        for (long long i = 0; i < n; ++i) {
            const char* e = std::strchr(p, '\n');
            std::string tok = e ? std::string(p, e - p) : std::string(p);
            vals.push_back(FloatValue::finite(rational_from_decimal(tok)));
            p = e ? e + 1 : p + tok.size();
        }
        ReductionPlan plan = ReductionPlan::balanced(n, g);
        plan.tree_combine = tree != 0;
        return put(fv_str(reduce_with_plan(vals, FloatFormat::of(kind_of(fmt)), plan)), out, cap);
    } catch (const std::exception& e) {
        put(std::string("error: ") + e.what(), out, cap);
        return 1;
    }
}

// Runs scenario_from_json + SimEngine::simulate + compute_metrics and returns
// a JSON document {metrics, wall_ns, events, transcripts, logical_progress}.
int ref_simulate_json(const char* scenario_json, char* out, long cap) {
    REF_GUARDED(out, cap, try {
        auto cfg = nlohmann::json::parse(scenario_json);
        Scenario s = scenario_from_json(cfg, ".");
        auto t0 = std::chrono::steady_clock::now();
        SimulationReport rep = SimEngine::simulate(s);
        auto t1 = std::chrono::steady_clock::now();
        MetricsReport m = compute_metrics(rep);
        nlohmann::ordered_json j;
        j["metrics"] = metrics_to_json(m);
        j["wall_ns"] = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
        j["events"] = rep.events_processed;
        j["kernels_completed"] = rep.kernels_completed;
        nlohmann::ordered_json tr;
        for (const auto& [vid, sigs] : rep.vctx_transcripts) {
            nlohmann::ordered_json arr = nlohmann::ordered_json::array();
            for (const auto& sig : sigs) arr.push_back({sig.semantic_id, sig.grid_size});
            tr[std::to_string(vid.value)] = arr;
        }
        j["transcripts"] = tr;
        nlohmann::ordered_json lp;
        for (const auto& [vid, p] : rep.logical_progress) lp[std::to_string(vid.value)] = p;
        j["logical_progress"] = lp;
        nlohmann::ordered_json pre = nlohmann::ordered_json::array();
        for (const auto& pr : rep.preemptions) {
            pre.push_back({{"vctx", pr.vctx.value},
                           {"pctx", pr.pctx.value},
                           {"signal", to_decimal_string(pr.signal_time)},
                           {"boundary_wait", to_decimal_string(pr.boundary_wait)},
                           {"overhead", to_decimal_string(pr.overhead)}});
        }
        j["preemptions"] = pre;
        j["policy_errors"] = rep.policy_errors;
        add_migrations(j, rep);
        return put(j.dump(), out, cap);
    } catch (const std::exception& e) {
        put(std::string("error: ") + e.what(), out, cap);
        return 1;
    });
}

// check_immutable_equivalence (equivalence.cpp:56-95)
int ref_equivalence_json(const char* scenario_json, char* out, long cap) {
    REF_GUARDED(out, cap, try {
        auto cfg = nlohmann::json::parse(scenario_json);
        Scenario s = scenario_from_json(cfg, ".");
        auto t0 = std::chrono::steady_clock::now();
        EquivalenceResult r = check_immutable_equivalence(s);
        auto t1 = std::chrono::steady_clock::now();
        nlohmann::ordered_json j;
        j["equivalent"] = r.equivalent;
        j["transcripts_match"] = r.transcripts_match;
        j["reductions_match"] = r.reductions_match;
        j["max_delta"] = numerator(r.max_delta).str() + "/" + denominator(r.max_delta).str();
        j["wall_ns"] = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
        return put(j.dump(), out, cap);
    } catch (const std::exception& e) {
        put(std::string("error: ") + e.what(), out, cap);
        return 1;
    });
}

// gen_poisson (which == 0) / gen_burst (which == 1) (trace.cpp:189-232) with a
// RequestTemplate (trace.hpp:41-53); returns the serialized JSONL trace
// (serialize_trace, trace.cpp:153-155).  rates[] = {rate, duration} or
// {base, burst, burst_duration, period, duration}.
int ref_gen_trace(int which, const double* rates, int kind, int prompt, int prompt_max, int output, int output_max,
                  int iterations, int streams, unsigned long long seed, char* out, long cap) {
    try {
        RequestTemplate t;
        t.kind = kind == 0 ? "inference" : "training";
        t.prompt_tokens = prompt;
        t.prompt_tokens_max = prompt_max;
        t.output_tokens = output;
        t.output_tokens_max = output_max;
        t.iterations = iterations;
        t.streams = streams;
        std::vector<RequestTraceRecord> recs =
            which == 0 ? gen_poisson(rates[0], rates[1], t, seed)
                       : gen_burst(rates[0], rates[1], rates[2], rates[3], rates[4], t, seed);
        std::ostringstream os;
        serialize_trace(recs, os);
        return put(os.str(), out, cap);
    } catch (const std::exception& e) {
        put(std::string("error: ") + e.what(), out, cap);
        return 1;
    }
}

// expand_workload (workload.cpp:51-174) of a JSONL trace with the given
// profile grids; returns one line per kernel: "job phase grid decode_index
// request seed" (seed = reduction seed, present when reduction_elements > 0).
int ref_expand(const char* trace_jsonl, long long tokens_per_grid_unit, long long decode_grid, long long train_grid,
               int default_iterations, char* out, long cap) {
    try {
        auto recs = parse_trace_string(trace_jsonl);
        WorkloadProfiles prof;
        prof.inference["default"].tokens_per_grid_unit = tokens_per_grid_unit;
        prof.inference["default"].decode_grid = decode_grid;
        prof.inference["default"].reduction_elements = 1;  // attach the lab seed to every kernel
        prof.training["default"].grid = train_grid;
        prof.training["default"].iterations = default_iterations;
        prof.training["default"].reduction_elements = 1;
        ExpandedWorkload w = expand_workload(recs, prof);
        std::ostringstream os;
        std::vector<std::string> lines;
        // emit in (request, position) order like the native expansion
        struct Row { long long req; std::size_t job, pos; const Kernel* k; };
        std::vector<Row> rows;
        for (std::size_t j = 0; j < w.jobs.size(); ++j)
            for (std::size_t i = 0; i < w.jobs[j].kernels.size(); ++i)
                rows.push_back({w.jobs[j].kernels[i].request.value, j, i, &w.jobs[j].kernels[i]});
        std::stable_sort(rows.begin(), rows.end(), [](const Row& a, const Row& b) {
            return a.req != b.req ? a.req < b.req : a.pos < b.pos;
        });
        for (const Row& r : rows) {
            const Kernel& k = *r.k;
            os << r.job << ' ' << static_cast<int>(k.phase) << ' ' << k.signature.grid_size << ' '
               << k.decode_index << ' ' << k.request.value << ' '
               << (k.reduction ? k.reduction->value_seed : 0ULL) << ' ' << to_decimal_string(k.arrival_floor) << '\n';
        }
        return put(os.str(), out, cap);
    } catch (const std::exception& e) {
        put(std::string("error: ") + e.what(), out, cap);
        return 1;
    }
}

// compute_migration_set / full_eager_set (migration.cpp:21-58) on a working
// set given as lines "id bytes dirty place,place,..." and touched region ids
// "id id ...".  Returns "eager ids | eager_bytes | lazy ids | lazy_bytes" or
// "error: <Errc>".
int ref_migration_set(const char* regions_nl, const char* touched_sp, int dst, int full, char* out, long cap) {
    try {
        VirtualContext v;
        std::istringstream rs(regions_nl);
        std::string line;
        while (std::getline(rs, line)) {
            if (line.empty()) continue;
            std::istringstream ls(line);
            long long id, bytes;
            int dirty;
            std::string places;
            ls >> id >> bytes >> dirty >> places;
            MemoryRegion r;
            r.id = RegionId(static_cast<std::int32_t>(id));
            r.bytes = static_cast<std::uint64_t>(bytes);
            r.dirty = dirty != 0;
            std::istringstream ps(places == "-" ? "" : places);
            std::string p;
            while (std::getline(ps, p, ',')) r.resident_on.insert(PctxId(std::stoi(p)));
            v.working_set[r.id] = r;
        }
        Kernel k;
        std::istringstream ts(touched_sp);
        long long t;
        while (ts >> t) k.touched_regions.push_back(RegionId(static_cast<std::int32_t>(t)));
        MigrationSet m = full ? full_eager_set(v) : compute_migration_set(v, k, PctxId(dst));
        std::ostringstream os;
        for (RegionId r : m.eager) os << r.value << ' ';
        os << "| " << m.eager_bytes << " | ";
        for (RegionId r : m.lazy) os << r.value << ' ';
        os << "| " << m.lazy_bytes;
        return put(os.str(), out, cap);
    } catch (const SimError& e) {
        put(std::string("error: ") + errc_name(e.code()), out, cap);
        return 0;
    } catch (const std::exception& e) {
        put(std::string("error: ") + e.what(), out, cap);
        return 1;
    }
}


// Every hook of a reference policy on one flat snapshot (oracle/policy_case.h):
// on_launch, on_congestion (pool_exhausted set), on_completion,
// launch_order_key, next_review_time, and predict_hol_blocking per pctx.
int ref_policy_eval(const pc_case* c, pc_result* out) {
    try {
        auto sig = [](int i) {
            return KernelSignature{PC_SIG_NAMES[(i / 2) % 4], (i & 1) ? 128 : 256};
        };
        auto R = [](long long x) { return Rational(x); };
        DurationPredictor pred(Rational(3, 10), R(c->cold_default));
        for (int i = 0; i < c->n_obs; ++i) pred.observe(sig(c->obs_sig[i]), R(c->obs_dur[i]));
        PolicyView v;
        v.now = R(c->now);
        v.predictor = &pred;
        v.active_vctx_count = c->active_vctx_count;
        for (int i = 0; i < c->n_p; ++i) {
            const pc_pctx& q = c->p[i];
            PolicyView::PctxEntry e;
            e.id = PctxId(i);
            e.device = DeviceId(q.device);
            e.tier = Rational(BigInt(q.tier_num), BigInt(q.tier_den));
            e.standby = q.standby != 0;
            if (q.bound >= 0) e.bound = VctxId(q.bound);
            e.available = q.available != 0;
            if (q.running_kernel >= 0) e.running_kernel = KernelId((std::int32_t)q.running_kernel);
            e.running_signature = sig(q.running_sig);
            e.running_remaining = R(q.running_remaining);
            e.running_phase = (Phase)q.running_phase;
            e.running_priority = (PriorityClass)q.running_priority;
            for (int k = 0; k < q.n_queued; ++k) e.queued.push_back({sig(q.queued_sig[k]), R(q.queued_hint[k])});
            v.pctxs.push_back(e);
        }
        for (const auto& e : v.pctxs) {  // as the engine's build_view (engine.cpp:345-365)
            if (e.bound) v.bound_tier_sums[e.device] += e.tier;
            auto it = v.min_tiers.find(e.device);
            if (it == v.min_tiers.end() || e.tier < it->second) v.min_tiers[e.device] = e.tier;
        }
        for (int i = 0; i < c->n_v; ++i) {
            const pc_vctx& q = c->v[i];
            PolicyView::VctxEntry e;
            e.id = VctxId(i);
            e.priority = (PriorityClass)q.priority;
            e.quarantined = q.quarantined != 0;
            e.bound = q.bound != 0;
            e.pending = q.pending;
            e.head_phase = (Phase)q.head_phase;
            e.decoding = q.decoding != 0;
            v.vctxs.push_back(e);
        }
        Kernel k;
        k.signature = sig(c->l_sig);
        k.base_duration = R(c->l_base);
        k.compute_saturation = Rational(BigInt(c->l_sat_num), BigInt(c->l_sat_den));
        k.phase = (Phase)c->l_phase;
        LaunchContext l;
        l.vctx = VctxId(c->l_vctx);
        if (c->l_has_kernel) l.kernel = &k;
        l.request_arrival = R(c->l_request_arrival);
        if (c->l_has_slo) l.slo = SloSpec{R(c->l_ttft), R(c->l_tpot), std::nullopt};
        PolicyConfig cfg;
        static const char* names[4] = {"slo-aware", "tpot-first", "temporal", "static"};
        cfg.name = names[c->policy];
        cfg.quantum = R(c->quantum);
        for (int i = 0; i < c->n_assign; ++i) cfg.assignments[VctxId(c->assign_v[i])] = PctxId(c->assign_p[i]);
        auto pol = make_policy(cfg);
        auto put_d = [](const PolicyDecision& d, int32_t* kind, int32_t* target) {
            *kind = (int32_t)d.kind;  // DispatchDirect, DispatchRemap, DispatchDefer, Preempt, NoAction
            *target = d.target.value;
        };
        put_d(pol->on_launch(v, l), &out->launch_kind, &out->launch_target);
        put_d(pol->on_completion(v, l), &out->completion_kind, &out->completion_target);
        LaunchContext lc = l;
        lc.pool_exhausted = true;
        put_d(pol->on_congestion(v, lc), &out->congestion_kind, &out->congestion_target);
        out->order_key = pol->launch_order_key(l);
        auto r = pol->next_review_time(v);
        out->has_review = r.has_value();
        auto to_i64 = [](const Rational& x) -> long long {
            // integral inputs keep every quantity integral; floor otherwise
            BigInt q = numerator(x) / denominator(x);
            return q.convert_to<long long>();
        };
        out->review = r ? to_i64(*r) : 0;
        for (int i = 0; i < c->n_p && i < PC_MAXP; ++i) out->hol[i] = to_i64(predict_hol_blocking(v, v.pctxs[i], pred));
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ref_policy_eval: %s\n", e.what());
        return 1;
    }
}

// The reference EWMA predictor (predictor.cpp:14-25) over n observations of
// one signature at alpha = an/ad: floor and ceil of the exact prediction.
int ref_predict_ewma(int n, const long long* durs, long long an, long long ad, long long* lo, long long* hi) {
    try {
        DurationPredictor p(Rational(BigInt(an), BigInt(ad)), Rational(1));
        KernelSignature sig{"k", 1};
        for (int i = 0; i < n; ++i) p.observe(sig, Rational(durs[i]));
        Rational x = p.predict(sig);
        BigInt q = numerator(x) / denominator(x);
        *lo = q.convert_to<long long>();
        *hi = (Rational(q) == x) ? *lo : *lo + 1;
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// compute_metrics (metrics.cpp:35-85) over request outcomes given as
// parallel arrays (integer times).  Output: "key num/den" lines, exact.
int ref_compute_metrics(long long n, const int* inference, const int* completed, const int* tokens,
                        const int* has_slo, const long long* arrival, const long long* first,
                        const long long* last, const long long* ttft_slo, const long long* tpot_slo,
                        const long long* kernels_done, long long makespan, long long kernels_completed, char* out,
                        long cap) {
    try {
        SimulationReport rep;
        rep.end_clock = Rational(makespan);
        rep.kernels_completed = kernels_completed;
        for (long long i = 0; i < n; ++i) {
            RequestOutcome r;
            r.meta.id = RequestId((std::int32_t)i);
            r.meta.arrival = Rational(arrival[i]);
            r.meta.inference = inference[i] != 0;
            r.meta.output_tokens = tokens[i];
            if (has_slo[i]) r.meta.slo = SloSpec{Rational(ttft_slo[i]), Rational(tpot_slo[i]), std::nullopt};
            r.completed = completed[i] != 0;
            r.first_decode_finish = Rational(first[i]);
            r.last_finish = Rational(last[i]);
            r.kernels_done = (int)kernels_done[i];
            rep.requests.push_back(r);
        }
        MetricsReport m = compute_metrics(rep);
        std::ostringstream os;
        auto q = [&](const char* k, const Rational& x) { os << k << ' ' << numerator(x).str() << '/' << denominator(x).str() << '\n'; };
        auto dist = [&](const char* k, const DistSummary& d) {
            os << k << "_count " << d.count << '\n';
            if (d.count == 0) return;
            std::string b(k);
            q((b + "_mean").c_str(), d.mean);
            q((b + "_p50").c_str(), d.p50);
            q((b + "_p90").c_str(), d.p90);
            q((b + "_p99").c_str(), d.p99);
        };
        os << "inference_completed " << m.inference_completed << '\n';
        os << "training_kernels_completed " << m.training_kernels_completed << '\n';
        os << "tpot_excluded " << m.tpot_excluded << '\n';
        os << "slo_requests " << m.slo_requests << '\n';
        os << "ttft_violations " << m.ttft_violations << '\n';
        os << "tpot_violations " << m.tpot_violations << '\n';
        q("inference_throughput", m.inference_throughput);
        q("training_throughput", m.training_throughput);
        q("ttft_violation_rate", m.ttft_violation_rate);
        q("tpot_violation_rate", m.tpot_violation_rate);
        dist("ttft", m.ttft);
        dist("tpot", m.tpot);
        return put(os.str(), out, cap);
    } catch (const std::exception& e) {
        put(std::string("error: ") + e.what(), out, cap);
        return 1;
    }
}

}  // extern "C"
