// The reference-named C++ façade (include/detshare/corosim.hpp) over the C ABI.
//
//   test_facade          host-only checks (no GPU): Rational, make_policy /
//                        policy_names, the built-ins through the C ABI, a user
//                        Policy through the vtable trampolines
//   test_facade gpu      the drop-in path on a B200: create_pool -> Device,
//                        bind errors, a user Policy injected
//                        into SimEngine (engine.hpp:155) that returns illegal
//                        decisions (Remap to a bound pctx ->
//                        PolicyError -> Defer), snapshot, ledger, exclusive_baseline
//
// Built and run by tests/test_facade.py (host part) and
// tests/test_gpu_boundary.py (gpu part), linked against libdetshare.so.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "detshare/corosim.hpp"

using namespace corosim;

static int failures = 0;
#define EXPECT(c)                                                          \
    do {                                                                   \
        if (!(c)) {                                                        \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);      \
            ++failures;                                                    \
        }                                                                  \
    } while (0)

// A reference-style user policy: the first `bad` launch decisions are
// illegal (Remap to a bound pctx, then to no pctx, then an unknown kind is
// impossible from C++ — a Preempt of self), after that the smallest free
// feasible tier, or Direct when bound.
class Adversarial : public Policy {
  public:
    explicit Adversarial(int bad) : bad_(bad) {}
    std::string_view name() const override { return "adversarial"; }
    PolicyDecision on_launch(const PolicyView& view, const LaunchContext& launch) const override {
        const auto* v = view.vctx(launch.vctx);
        if (calls_++ < bad_) {
            for (const auto& p : view.pctxs)
                if (p.bound && *p.bound != launch.vctx) return PolicyDecision::remap(p.id);  // bound pctx
            return PolicyDecision::remap(PctxId(999));                                      // unknown pctx
        }
        if (v && v->bound) return PolicyDecision::direct();
        const PolicyView::PctxEntry* best = nullptr;
        for (const auto& p : view.pctxs)
            if (!p.bound && p.available && view.feasible_bind(p) && (!best || p.tier < best->tier)) best = &p;
        return best ? PolicyDecision::remap(best->id) : PolicyDecision::defer();
    }
    int launch_order_key(const LaunchContext& launch) const override {
        return launch.kernel && launch.kernel->phase == Phase::Decode ? 0 : 1;
    }
    mutable int calls_ = 0;

  private:
    int bad_;
};

static void host_tests() {
    // Rational (rational.hpp): exact, normalised
    Rational a(1, 4), b(2, 8), c(3, 4);
    EXPECT(a == b);
    EXPECT(a + c == Rational(1));
    EXPECT(c - a == Rational(1, 2));
    EXPECT(a * c == Rational(3, 16));
    EXPECT(c / a == Rational(3));
    EXPECT(Rational(-7, 2).floor_ns() == -4);
    EXPECT(Rational(1, 3) < Rational(1, 2));
    // policies (policies.hpp:74-75)
    auto names = policy_names();
    EXPECT(names.size() >= 4);
    bool threw = false;
    try {
        make_policy(PolicyConfig{"no-such-policy"});
    } catch (const SimError& e) {
        threw = e.code() == Errc::ConfigError;
    }
    EXPECT(threw);
    // TPOT-First through the C ABI: a decode launch is served first; an unbound
    // vctx with a free full tier is remapped there
    auto tpot = make_policy(PolicyConfig{"tpot-first"});
    EXPECT(tpot->name() == "tpot-first");
    PolicyView v;
    v.now = Rational(1000);
    for (int i = 0; i < 2; ++i) {
        PolicyView::PctxEntry p;
        p.id = PctxId(i);
        p.device = DeviceId(0);
        p.tier = i == 0 ? Rational(1, 4) : Rational(1);
        v.pctxs.push_back(p);
    }
    v.bound_tier_sums[DeviceId(0)] = Rational(0);
    v.min_tiers[DeviceId(0)] = Rational(1, 4);
    PolicyView::VctxEntry x;
    x.id = VctxId(0);
    x.priority = PriorityClass::LatencyCritical;
    x.pending = 1;
    x.head_phase = Phase::Decode;
    x.decoding = true;
    v.vctxs.push_back(x);
    v.active_vctx_count = 1;
    Kernel k;
    k.id = KernelId(0);
    k.vctx = VctxId(0);
    k.signature = KernelSignature{"decode/step", 163};
    k.base_duration = Rational(4000000);
    k.compute_saturation = Rational(1, 2);
    k.phase = Phase::Decode;
    LaunchContext l;
    l.vctx = VctxId(0);
    l.kernel = &k;
    l.slo = SloSpec{Rational(100000000), Rational(40000000), std::nullopt};
    EXPECT(tpot->launch_order_key(l) == 0);
    PolicyDecision d = tpot->on_launch(v, l);
    EXPECT(d.kind == PolicyDecision::Kind::DispatchRemap);
    EXPECT(d.target == PctxId(1));  // saturation 1/2, fair share 1: the smallest tier >= 1/2 is the full one
    k.phase = Phase::Prefill;
    EXPECT(tpot->launch_order_key(l) == 2);
    // a user policy through the C vtable trampolines (what the engine calls)
    Adversarial adv(1);
    ds_view cv;
    std::vector<std::string> keep;
    detail::to_c(v, cv, keep);
    ds_launch_ctx cl;
    k.phase = Phase::Decode;
    detail::to_c(l, cl);
    ds_decision d1, d2;
    detail::on_launch_tr(&adv, &cv, &cl, &d1);  // first: illegal remap to an unknown pctx
    EXPECT(d1.kind == (int)PolicyDecision::Kind::DispatchRemap && d1.target == 999);
    detail::on_launch_tr(&adv, &cv, &cl, &d2);  // then the smallest free feasible tier
    EXPECT(d2.kind == (int)PolicyDecision::Kind::DispatchRemap && d2.target == 0);
    EXPECT(detail::order_key_tr(&adv, &cl) == 0);
    // predict_hol_blocking over the C view: nothing running -> 0
    std::int64_t hol = -1;
    EXPECT(ds_predict_hol_blocking(&cv, 1, &hol) == DS_OK && hol == 0);
    std::printf("host facade tests: %s\n", failures ? "FAILED" : "ok");
}

static void gpu_tests() {
    // create_pool (types.cpp:87-106) -> Device; an out-of-range tier is InvalidTier
    bool threw = false;
    try {
        Device bad(0, {Rational(3, 2)});
    } catch (const SimError& e) {
        threw = e.code() == Errc::InvalidTier;
    }
    EXPECT(threw);
    Device dev(0, {Rational(1, 4), Rational(1, 2), Rational(1)});
    EXPECT(dev.pctx_count() == 3);
    VctxId t0 = dev.add_tenant("decode", PriorityClass::LatencyCritical);
    VctxId t1 = dev.add_tenant("train", PriorityClass::BestEffort);
    void* out = nullptr;
    check(ds_ipc_alloc(0, 3 * 8 * 4096, &out));
    struct {
        std::uint64_t out, ns;
    } spin{(std::uint64_t)out, 20000};
    int ks = dev.add_kernel("spin", DS_BODY_SPIN, 296, 1, 1, &spin, sizeof spin, Phase::Decode);
    dev.start();
    // bind script: BindConflict, DoubleBind, rebind after unbind
    bind(dev, t0, PctxId(0));
    threw = false;
    try {
        bind(dev, t1, PctxId(0));
    } catch (const SimError& e) {
        threw = e.code() == Errc::BindConflict;
    }
    EXPECT(threw);
    threw = false;
    try {
        bind(dev, t0, PctxId(1));
    } catch (const SimError& e) {
        threw = e.code() == Errc::DoubleBind;
    }
    EXPECT(threw);
    unbind(dev, t0);
    bind(dev, t0, PctxId(1));
    unbind(dev, t0);
    // a user policy injected into the engine: its first 4 decisions are illegal
    auto* adv = new Adversarial(4);
    EngineConfig ec;
    SimEngine eng(dev, ec, std::unique_ptr<Policy>(adv));
    int j0 = eng.add_job(t0, PriorityClass::LatencyCritical);
    int j1 = eng.add_job(t1, PriorityClass::BestEffort);
    eng.start();
    RecordSpec r;
    r.semantic_id = "spin";
    r.grid_size = 296;
    r.kernels = {ks, ks};
    r.phase = Phase::Decode;
    r.base_hint = Rational(100000);
    r.compute_saturation = Rational(1, 2);
    KernelId last0, last1;
    for (int i = 0; i < 3; ++i) last0 = eng.submit(j0, r);
    r.phase = Phase::Training;
    for (int i = 0; i < 3; ++i) last1 = eng.submit(j1, r);
    eng.wait(last0, 30000);
    eng.wait(last1, 30000);
    PolicyView snap = eng.snapshot();
    EXPECT(snap.pctxs.size() == 3);
    EXPECT(snap.vctxs.size() == 2);
    EngineCounters ctr = eng.counters();
    std::printf("engine counters: decisions %llu dispatches %llu completed %llu policy_errors %llu\n",
                (unsigned long long)ctr.decisions, (unsigned long long)ctr.dispatches,
                (unsigned long long)ctr.completed, (unsigned long long)ctr.policy_errors);
    EXPECT(ctr.policy_errors == 4);  // every illegal decision became Defer + PolicyError
    EXPECT(ctr.completed == 6);
    eng.stop();  // finalize: records and device kernels unchanged (no DS_RECORD_MUTATED)
    ds_ledger led;
    check(ds_ledger_get(dev.handle(), &led));
    std::printf("ledger: switches %llu grants %llu\n", (unsigned long long)led.ctx_switches,
                (unsigned long long)led.migrations);
    dev.stop();
    // exclusive_baseline: the same kernel as a plain grid (executor stopped: it owns every SM)
    exclusive_baseline(dev, ks, nullptr);
    ds_ipc_free(0, out);
    std::printf("gpu facade tests: %s\n", failures ? "FAILED" : "ok");
}

int main(int argc, char** argv) {
    try {
        host_tests();
        if (argc > 1 && std::strcmp(argv[1], "gpu") == 0) gpu_tests();
    } catch (const std::exception& e) {
        std::printf("EXCEPTION %s\n", e.what());
        return 1;
    }
    return failures ? 1 : 0;
}
