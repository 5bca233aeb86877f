// User policies over the C ABI: the reference's Policy virtuals
// (proj/include/corosim/policy/policy.hpp:97-126) as a POD vtable of hooks
// over a C snapshot of PolicyView (policy.hpp:24-69).  AbiPolicy adapts a
// vtable to the engine's Policy interface; the engine validates whatever it
// returns (engine.cpp apply(), the reference's apply_decision
// engine.cpp:688-754), so an illegal decision from user code degrades to
// Defer and counts a policy error.
#include <cstring>
#include <memory>
#include <string>

#include "../../include/detshare/ds.h"
#include "policy.hpp"

namespace detshare {

namespace {

void to_c_launch(const LaunchContext& lc, ds_launch_ctx* o) {
    std::memset(o, 0, sizeof(*o));
    o->vctx = lc.vctx;
    o->request_arrival_ns = lc.request_arrival;
    o->pool_exhausted = lc.pool_exhausted ? 1 : 0;
    if (lc.slo) {
        o->has_slo = 1;
        o->ttft_ns = lc.slo->ttft_deadline;
        o->tpot_ns = lc.slo->tpot_deadline;
    }
    o->request = -1;
    o->decode_index = -1;
    o->phase = (int32_t)Phase::Other;
    o->sat_num = o->sat_den = 1;
    if (lc.kernel) {
        const LaunchRecord& k = *lc.kernel;
        o->has_kernel = 1;
        o->kernel_id = k.id;
        o->semantic_id = k.signature.semantic_id.c_str();
        o->grid_size = k.signature.grid_size;
        o->base_hint_ns = k.base_duration;
        o->sat_num = k.compute_saturation.num;
        o->sat_den = k.compute_saturation.den;
        o->phase = (int32_t)k.phase;
        o->decode_index = k.decode_index;
        o->request = k.request;
        o->arrival_ns = k.arrival;
    }
}

ds_decision to_c(const PolicyDecision& d) { return ds_decision{(int32_t)d.kind, d.target}; }

PolicyDecision from_c(const ds_decision& d) {
    // an out-of-range kind is an illegal decision: the engine rejects a remap to no pctx (policy error)
    if (d.kind < 0 || d.kind > (int)PolicyDecision::Kind::NoAction) return PolicyDecision::remap(-1);
    return PolicyDecision{(PolicyDecision::Kind)d.kind, d.target};
}

class AbiPolicy : public Policy {
  public:
    AbiPolicy(const ds_policy_vtable& vt, void* user) : vt_(vt), user_(user), name_(vt.name ? vt.name : "user") {}
    ~AbiPolicy() override {
        if (vt_.destroy) vt_.destroy(user_);
    }
    std::string_view name() const override { return name_; }
    PolicyDecision on_launch(const PolicyView& view, const LaunchContext& launch) const override {
        return call(vt_.on_launch, view, launch, PolicyDecision::defer());
    }
    PolicyDecision on_completion(const PolicyView& view, const LaunchContext& next) const override {
        return call(vt_.on_completion, view, next, PolicyDecision::no_action());
    }
    PolicyDecision on_congestion(const PolicyView& view, const LaunchContext& launch) const override {
        return call(vt_.on_congestion, view, launch, PolicyDecision::defer());
    }
    int launch_order_key(const LaunchContext& launch) const override {
        if (!vt_.launch_order_key) return 0;
        ds_launch_ctx c;
        to_c_launch(launch, &c);
        return vt_.launch_order_key(user_, &c);
    }
    std::optional<Time> next_review_time(const PolicyView& view) const override {
        if (!vt_.next_review_time) return std::nullopt;
        auto v = std::make_unique<ds_view>();
        view_to_c(view, v.get());
        int64_t t = 0;
        if (!vt_.next_review_time(user_, v.get(), &t)) return std::nullopt;
        return t;
    }

  private:
    using Hook = void (*)(void*, const ds_view*, const ds_launch_ctx*, ds_decision*);
    PolicyDecision call(Hook h, const PolicyView& view, const LaunchContext& launch, PolicyDecision dflt) const {
        if (!h) return dflt;
        auto v = std::make_unique<ds_view>();
        view_to_c(view, v.get());
        ds_launch_ctx c;
        to_c_launch(launch, &c);
        ds_decision d = to_c(dflt);
        h(user_, v.get(), &c, &d);
        return from_c(d);
    }
    ds_policy_vtable vt_;
    void* user_;
    std::string name_;
};

}  // namespace

void view_to_c(const PolicyView& v, ds_view* o) {
    std::memset(o, 0, sizeof(*o));
    o->now_ns = v.now;
    o->n_pctx = (int32_t)std::min<size_t>(v.pctxs.size(), DS_VIEW_MAX_PCTX);
    for (int i = 0; i < o->n_pctx; ++i) {
        const auto& p = v.pctxs[i];
        ds_view_pctx& c = o->pctx[i];
        c.id = p.id;
        c.device = p.device;
        c.tier_num = p.tier.num;
        c.tier_den = p.tier.den;
        c.standby = p.standby;
        c.available = p.available;
        c.bound = p.bound ? *p.bound : -1;
        c.has_running = p.running_kernel ? 1 : 0;
        c.running_kernel = p.running_kernel ? *p.running_kernel : 0;
        c.running_semantic_id = p.running_signature.semantic_id.c_str();
        c.running_grid = p.running_signature.grid_size;
        c.running_remaining_ns = p.running_remaining;
        c.running_phase = (int32_t)p.running_phase;
        c.running_priority = (int32_t)p.running_priority;
    }
    o->n_vctx = (int32_t)std::min<size_t>(v.vctxs.size(), DS_VIEW_MAX_VCTX);
    for (int i = 0; i < o->n_vctx; ++i) {
        const auto& x = v.vctxs[i];
        ds_view_vctx& c = o->vctx[i];
        c.id = x.id;
        c.priority = (int32_t)x.priority;
        c.quarantined = x.quarantined;
        c.bound = x.bound;
        c.pending = x.pending;
        c.head_phase = (int32_t)x.head_phase;
        c.decoding = x.decoding;
    }
    int nd = 0;
    for (const auto& [dev, f] : v.bound_tier_sums) nd = std::max(nd, dev + 1);
    for (const auto& [dev, f] : v.min_tiers) nd = std::max(nd, dev + 1);
    o->n_devices = std::min(nd, DS_VIEW_MAX_DEVICES);
    for (int d = 0; d < o->n_devices; ++d) {
        auto b = v.bound_tier_sums.find(d);
        o->bound_tier_sum_num[d] = b == v.bound_tier_sums.end() ? 0 : b->second.num;
        o->bound_tier_sum_den[d] = b == v.bound_tier_sums.end() ? 1 : b->second.den;
        auto m = v.min_tiers.find(d);
        o->min_tier_num[d] = m == v.min_tiers.end() ? 1 : m->second.num;
        o->min_tier_den[d] = m == v.min_tiers.end() ? 1 : m->second.den;
    }
    o->active_vctx_count = v.active_vctx_count;
    o->predictor = v.predictor;
}

void view_from_c(const ds_view& o, PolicyView& v, const DurationPredictor* fallback) {
    v = PolicyView{};
    v.now = o.now_ns;
    for (int i = 0; i < o.n_pctx && i < DS_VIEW_MAX_PCTX; ++i) {
        const ds_view_pctx& c = o.pctx[i];
        PolicyView::PctxEntry p;
        p.id = c.id;
        p.device = c.device;
        p.tier = Frac{c.tier_num, c.tier_den};
        p.standby = c.standby != 0;
        p.available = c.available != 0;
        if (c.bound >= 0) p.bound = c.bound;
        if (c.has_running) p.running_kernel = c.running_kernel;
        p.running_signature = KernelSignature{c.running_semantic_id ? c.running_semantic_id : "", c.running_grid};
        p.running_remaining = c.running_remaining_ns;
        p.running_phase = (Phase)c.running_phase;
        p.running_priority = (PriorityClass)c.running_priority;
        v.pctxs.push_back(p);
    }
    for (int i = 0; i < o.n_vctx && i < DS_VIEW_MAX_VCTX; ++i) {
        const ds_view_vctx& c = o.vctx[i];
        PolicyView::VctxEntry x;
        x.id = c.id;
        x.priority = (PriorityClass)c.priority;
        x.quarantined = c.quarantined != 0;
        x.bound = c.bound != 0;
        x.pending = c.pending;
        x.head_phase = (Phase)c.head_phase;
        x.decoding = c.decoding != 0;
        v.vctxs.push_back(x);
    }
    for (int d = 0; d < o.n_devices && d < DS_VIEW_MAX_DEVICES; ++d) {
        v.bound_tier_sums[d] = Frac{o.bound_tier_sum_num[d], o.bound_tier_sum_den[d]};
        v.min_tiers[d] = Frac{o.min_tier_num[d], o.min_tier_den[d]};
    }
    v.active_vctx_count = o.active_vctx_count;
    v.predictor = o.predictor ? static_cast<const DurationPredictor*>(o.predictor) : fallback;
}

void launch_from_c(const ds_launch_ctx& c, LaunchRecord& rec, LaunchContext& lc) {
    lc = LaunchContext{};
    lc.vctx = c.vctx;
    lc.request_arrival = c.request_arrival_ns;
    lc.pool_exhausted = c.pool_exhausted != 0;
    if (c.has_slo) lc.slo = SloSpec{c.ttft_ns, c.tpot_ns};
    if (c.has_kernel) {
        rec = LaunchRecord{};
        rec.id = c.kernel_id;
        rec.job = c.vctx;
        rec.signature = KernelSignature{c.semantic_id ? c.semantic_id : "", c.grid_size};
        rec.base_duration = c.base_hint_ns;
        rec.compute_saturation = Frac{c.sat_num, c.sat_den};
        rec.phase = (Phase)c.phase;
        rec.request = c.request;
        rec.decode_index = c.decode_index;
        rec.slo = lc.slo;
        rec.arrival = c.arrival_ns;
        rec.request_arrival = c.request_arrival_ns;
        lc.kernel = &rec;
    }
}

std::unique_ptr<Policy> make_abi_policy(const ds_policy_vtable& vt, void* user) {
    return std::make_unique<AbiPolicy>(vt, user);
}

}  // namespace detshare

using namespace detshare;

extern "C" {

int ds_predictor_predict(const void* predictor, const char* semantic_id, int64_t grid, int has_hint, int64_t hint_ns,
                         int64_t* out_ns) {
    if (!predictor || !out_ns) return DS_INVALID_ARGUMENT;
    const auto* p = static_cast<const DurationPredictor*>(predictor);
    KernelSignature sig{semantic_id ? semantic_id : "", grid};
    *out_ns = has_hint ? p->predict(sig, hint_ns) : p->predict(sig);
    return DS_OK;
}

int ds_predict_hol_blocking(const ds_view* view, int pctx, int64_t* out_ns) {
    if (!view || !out_ns) return DS_INVALID_ARGUMENT;
    static const DurationPredictor dflt;
    PolicyView v;
    view_from_c(*view, v, &dflt);
    const auto* p = v.pctx(pctx);
    if (!p) return DS_INVALID_ARGUMENT;
    *out_ns = predict_hol_blocking(v, *p, *v.predictor);
    return DS_OK;
}

int ds_builtin_decide(const char* policy, int hook, const ds_view* view, const ds_launch_ctx* launch,
                      int64_t quantum_ns, ds_decision* out) {
    if (!policy || !view || !launch || !out || hook < 0 || hook > 3) return DS_INVALID_ARGUMENT;
    PolicyConfig cfg;
    cfg.name = policy;
    if (quantum_ns > 0) cfg.quantum = quantum_ns;
    std::unique_ptr<Policy> p;
    try {
        p = make_policy(cfg);
    } catch (const std::exception&) {
        return DS_CONFIG_ERROR;
    }
    static const DurationPredictor dflt;
    PolicyView v;
    view_from_c(*view, v, &dflt);
    LaunchRecord rec;
    LaunchContext lc;
    launch_from_c(*launch, rec, lc);
    if (hook == 3) {
        *out = ds_decision{DS_NO_ACTION, p->launch_order_key(lc)};
        return DS_OK;
    }
    PolicyDecision d = hook == 0 ? p->on_launch(v, lc) : hook == 1 ? p->on_completion(v, lc) : p->on_congestion(v, lc);
    *out = to_c(d);
    return DS_OK;
}

}  // extern "C"
