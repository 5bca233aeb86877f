// Host-side policy logic (csrc/policy.cpp) against the reference's decision
// rules and SPEC examples.  Built and run by tests/test_policy_cpp.py (no GPU).
#include <cassert>
#include <cstdio>
#include <stdexcept>

#include "../../paper_2603_15042_b200/csrc/policy.hpp"

using namespace detshare;

static int failures = 0;
#define CHECK(c)                                                   \
    do {                                                           \
        if (!(c)) {                                                \
            std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                            \
        }                                                          \
    } while (0)

static PolicyView::PctxEntry pctx(int id, Frac tier, std::optional<int> bound = std::nullopt) {
    PolicyView::PctxEntry p;
    p.id = id;
    p.tier = tier;
    p.bound = bound;
    return p;
}
static PolicyView::VctxEntry vctx(int id, PriorityClass pr, bool bound, int64_t pending = 1) {
    PolicyView::VctxEntry v;
    v.id = id;
    v.priority = pr;
    v.bound = bound;
    v.pending = pending;
    return v;
}

int main() {
    // Frac arithmetic (exact tiers)
    CHECK((Frac{1, 4} + Frac{3, 4}) == (Frac{1, 1}));
    CHECK((Frac{1, 3} < Frac{1, 2}));
    CHECK(!(Frac{2, 4} < Frac{1, 2}));

    // SPEC.md:303 EWMA {8, 12}, alpha 1/2 -> 10; cold start: hint, then max-by-semantic, then default
    {
        DurationPredictor p(0.5, 777);
        KernelSignature s{"k", 4};
        CHECK(p.predict(s) == 777);
        CHECK(p.predict(s, Time(5)) == 5);
        p.observe(s, 8);
        p.observe(s, 12);
        CHECK(p.predict(s) == 10);
        CHECK(p.predict(KernelSignature{"k", 9}) == 12);  // max seen for the semantic id
    }
    // SPEC.md:302 HOL blocking: running remainder 6 + queued predicted 5 = 11
    {
        DurationPredictor pred(0.3, 5);
        PolicyView v;
        auto p = pctx(0, Frac{1, 1}, 0);
        p.running_kernel = 1;
        p.running_remaining = 6;
        p.queued.push_back({KernelSignature{"q", 1}, 5});
        CHECK(predict_hol_blocking(v, p, pred) == 11);
    }
    // TPOT-First launch order: decode 0, other 1, prefill 2 (policies.cpp:216-222)
    {
        TpotFirstPolicy tf;
        LaunchRecord d, pf, tr;
        d.phase = Phase::Decode;
        pf.phase = Phase::Prefill;
        tr.phase = Phase::Training;
        LaunchContext l;
        l.kernel = &d;
        CHECK(tf.launch_order_key(l) == 0);
        l.kernel = &tr;
        CHECK(tf.launch_order_key(l) == 1);
        l.kernel = &pf;
        CHECK(tf.launch_order_key(l) == 2);
    }
    // placement: smallest free feasible tier >= min(saturation, fair share)
    {
        DurationPredictor pred;
        PolicyView v;
        v.predictor = &pred;
        v.pctxs = {pctx(0, {1, 4}), pctx(1, {3, 4}), pctx(2, {1, 1})};
        v.bound_tier_sums[0] = Frac{0, 1};
        v.min_tiers[0] = Frac{1, 4};
        v.vctxs = {vctx(0, PriorityClass::LatencyCritical, false), vctx(1, PriorityClass::BestEffort, false)};
        v.active_vctx_count = 2;
        LaunchRecord k;
        k.phase = Phase::Decode;
        k.compute_saturation = Frac{1, 1};
        LaunchContext l;
        l.vctx = 0;
        l.kernel = &k;
        SloAwarePolicy sa;
        auto d = sa.on_launch(v, l);
        CHECK(d.kind == PolicyDecision::Kind::DispatchRemap && d.target == 1);  // want 1/2 -> 3/4
        k.compute_saturation = Frac{1, 4};
        d = sa.on_launch(v, l);
        CHECK(d.kind == PolicyDecision::Kind::DispatchRemap && d.target == 0);  // want 1/4
    }
    // congestion: a latency-critical launch preempts the best-effort holder with the
    // largest remaining time; best-effort launchers never preempt
    {
        DurationPredictor pred;
        PolicyView v;
        v.predictor = &pred;
        auto a = pctx(0, {1, 2}, 1);
        a.running_kernel = 7;
        a.running_remaining = 10;
        auto b = pctx(1, {1, 2}, 2);
        b.running_kernel = 8;
        b.running_remaining = 30;
        v.pctxs = {a, b};
        v.bound_tier_sums[0] = Frac{1, 1};
        v.min_tiers[0] = Frac{1, 2};
        v.vctxs = {vctx(0, PriorityClass::LatencyCritical, false), vctx(1, PriorityClass::BestEffort, true),
                   vctx(2, PriorityClass::BestEffort, true)};
        v.active_vctx_count = 3;
        LaunchRecord k;
        k.phase = Phase::Decode;
        LaunchContext l;
        l.vctx = 0;
        l.kernel = &k;
        SloAwarePolicy sa;
        auto d = sa.on_congestion(v, l);
        CHECK(d.kind == PolicyDecision::Kind::Preempt && d.target == 1);
        l.vctx = 1;
        d = sa.on_congestion(v, l);
        CHECK(d.kind == PolicyDecision::Kind::DispatchDefer);
        // TPOT-First spares a decode victim when the launcher is a prefill
        v.pctxs[1].running_phase = Phase::Decode;
        k.phase = Phase::Prefill;
        l.vctx = 0;
        TpotFirstPolicy tf;
        d = tf.on_congestion(v, l);
        CHECK(d.kind == PolicyDecision::Kind::Preempt && d.target == 0);
    }
    // TPOT-First prefill admission: step_estimate * (active_decode + 1) > tpot -> defer
    {
        DurationPredictor pred(0.3, 1000);
        PolicyView v;
        v.predictor = &pred;
        auto a = pctx(0, {1, 2}, 1);
        a.running_kernel = 3;
        a.running_phase = Phase::Decode;
        a.running_signature = KernelSignature{"decode", 8};
        pred.observe(a.running_signature, 40);
        v.pctxs = {a, pctx(1, {1, 2})};
        v.bound_tier_sums[0] = Frac{1, 2};
        v.min_tiers[0] = Frac{1, 2};
        v.vctxs = {vctx(0, PriorityClass::LatencyCritical, false), vctx(1, PriorityClass::LatencyCritical, true)};
        v.active_vctx_count = 2;
        LaunchRecord k;
        k.phase = Phase::Prefill;
        LaunchContext l;
        l.vctx = 0;
        l.kernel = &k;
        l.slo = SloSpec{1000, 50};
        TpotFirstPolicy tf;
        CHECK(tf.on_launch(v, l).kind == PolicyDecision::Kind::DispatchDefer);  // 40 * 2 > 50
        l.slo = SloSpec{1000, 100};
        CHECK(tf.on_launch(v, l).kind == PolicyDecision::Kind::DispatchRemap);  // 80 <= 100
    }
    // temporal: owner = active[floor(now/quantum) % n]; review at the next boundary
    {
        TemporalBaselinePolicy tp(5);
        PolicyView v;
        v.vctxs = {vctx(0, PriorityClass::BestEffort, false), vctx(1, PriorityClass::BestEffort, false),
                   vctx(2, PriorityClass::BestEffort, false, 0)};
        v.now = 12;
        CHECK(tp.owner_at(v) == 0);  // slot 2 % 2 active
        v.now = 7;
        CHECK(tp.owner_at(v) == 1);
        CHECK(tp.next_review_time(v) == 10);
        v.pctxs = {pctx(0, {1, 2}), pctx(1, {1, 1})};
        v.bound_tier_sums[0] = Frac{0, 1};
        LaunchContext l;
        LaunchRecord k;
        l.kernel = &k;
        l.vctx = 1;
        auto d = tp.on_launch(v, l);
        CHECK(d.kind == PolicyDecision::Kind::DispatchRemap && d.target == 1);  // the full tier
        l.vctx = 0;
        CHECK(tp.on_launch(v, l).kind == PolicyDecision::Kind::DispatchDefer);
    }
    // static partition and make_policy
    {
        StaticPartitionPolicy sp({{0, 1}});
        PolicyView v;
        v.pctxs = {pctx(0, {1, 2}), pctx(1, {1, 2})};
        v.bound_tier_sums[0] = Frac{0, 1};
        v.vctxs = {vctx(0, PriorityClass::BestEffort, false)};
        LaunchContext l;
        LaunchRecord k;
        l.kernel = &k;
        l.vctx = 0;
        auto d = sp.on_launch(v, l);
        CHECK(d.kind == PolicyDecision::Kind::DispatchRemap && d.target == 1);
        bool threw = false;
        try {
            make_policy(PolicyConfig{"nope"});
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        CHECK(make_policy(PolicyConfig{"tpot-first"})->name() == "tpot-first");
        CHECK(policy_names().size() == 4);
    }
    if (failures) return 1;
    std::printf("policy tests ok\n");
    return 0;
}
