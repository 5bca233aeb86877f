// corosim.hpp — header-only C++ façade with the reference's names over the
// detshare C ABI (ds.h).  A caller of the reference library
// (/root/reference/proj/include/corosim/...) switches by including this
// header and linking libdetshare.so:
//
//   reference (corosim)                       here (same names)
//   Errc, SimError        errors.hpp:8-32     Errc, SimError (ds_status 1..10 + runtime codes)
//   Rational              rational.hpp:14-35  Rational: exact int64 fraction; times are ns
//   Id<Tag> / VctxId ...  ids.hpp:11-26       Id<Tag> / VctxId, PctxId, KernelId, DeviceId, RequestId
//   Phase, PriorityClass, KernelSignature     core/types.hpp:23-34
//   Kernel                core/types.hpp:46-68 (the policy-visible fields of a launch record)
//   SloSpec, PolicyView, LaunchContext, PolicyDecision, Policy   policy/policy.hpp:17-126
//   DurationPredictor::predict                policy/predictor.hpp:14-31 (the engine's predictor)
//   predict_hol_blocking                      policy/policy.hpp:92-95
//   PolicyConfig, make_policy, policy_names   policy/policies.hpp:12-75
//   SloAwarePolicy, TpotFirstPolicy, TemporalBaselinePolicy, StaticPartitionPolicy
//   create_pool -> Device, bind, unbind       core/types.hpp:130-137
//   SimEngine(…, std::unique_ptr<Policy>)     engine/engine.hpp:152-170
//   exclusive_baseline -> exclusive_baseline(Device&, kernel, stream): the plain-grid solo launch
//
// What changes: the engine drives real SMs of one B200 through the
// persistent coroutine executor instead of a performance model, so a
// SimEngine runs over a Device (a GPU sharing domain) whose tenants and
// device kernels are registered first, and records are submitted as they
// arrive instead of being read from a Scenario file.  Policies are unchanged:
// a user Policy subclass is handed to the engine through a POD vtable
// (ds_engine_create_with_policy) and sees the same PolicyView.
#pragma once

#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "ds.h"

namespace corosim {

// ---------------------------------------------------------------- errors
enum class Errc {  // errors.hpp:8-19 (ds_status 1..10, same order)
    InvalidTier,
    BindConflict,
    DoubleBind,
    CausalityViolation,
    EventBudgetExceeded,
    TraceViolation,
    PlanMismatch,
    InvalidSplit,
    ParseError,
    ConfigError,
};

inline const char* errc_name(Errc code) { return ds_status_name((int)code + 1); }

class SimError : public std::runtime_error {
  public:
    SimError(int status, const std::string& what)
        : std::runtime_error(std::string(ds_status_name(status)) + ": " + what), status_(status) {}
    // Errc for the reference's codes; runtime conditions (CUDA, timeouts,
    // failed tenants: status >= 100) map to ConfigError with status() kept
    Errc code() const { return status_ >= 1 && status_ <= 10 ? (Errc)(status_ - 1) : Errc::ConfigError; }
    int status() const { return status_; }

  private:
    int status_;
};

inline void check(int status) {
    if (status) throw SimError(status, ds_last_error());
}
inline void check_engine(int status) {
    if (status) throw SimError(status, ds_engine_last_error());
}

// ---------------------------------------------------------------- Rational
// Exact fraction over int64 (the reference uses Boost cpp_rational).  Times
// are integer nanoseconds on the engine clock.
class Rational {
  public:
    Rational(std::int64_t v = 0) : n_(v), d_(1) {}  // NOLINT (implicit, as cpp_rational)
    Rational(std::int64_t n, std::int64_t d) : n_(n), d_(d) {
        if (d_ == 0) throw std::domain_error("Rational: zero denominator");
        norm();
    }
    std::int64_t num() const { return n_; }
    std::int64_t den() const { return d_; }
    friend Rational operator+(const Rational& a, const Rational& b) {
        return from128((__int128)a.n_ * b.d_ + (__int128)b.n_ * a.d_, (__int128)a.d_ * b.d_);
    }
    friend Rational operator-(const Rational& a, const Rational& b) {
        return from128((__int128)a.n_ * b.d_ - (__int128)b.n_ * a.d_, (__int128)a.d_ * b.d_);
    }
    friend Rational operator*(const Rational& a, const Rational& b) {
        return from128((__int128)a.n_ * b.n_, (__int128)a.d_ * b.d_);
    }
    friend Rational operator/(const Rational& a, const Rational& b) {
        if (b.n_ == 0) throw std::domain_error("Rational: division by zero");
        return from128((__int128)a.n_ * b.d_, (__int128)a.d_ * b.n_);
    }
    Rational operator-() const { return Rational(-n_, d_); }
    Rational& operator+=(const Rational& o) { return *this = *this + o; }
    Rational& operator-=(const Rational& o) { return *this = *this - o; }
    friend bool operator==(const Rational& a, const Rational& b) { return a.n_ == b.n_ && a.d_ == b.d_; }
    friend bool operator!=(const Rational& a, const Rational& b) { return !(a == b); }
    friend bool operator<(const Rational& a, const Rational& b) { return (__int128)a.n_ * b.d_ < (__int128)b.n_ * a.d_; }
    friend bool operator>(const Rational& a, const Rational& b) { return b < a; }
    friend bool operator<=(const Rational& a, const Rational& b) { return !(b < a); }
    friend bool operator>=(const Rational& a, const Rational& b) { return !(a < b); }
    // floor to integer nanoseconds (the engine clock's resolution)
    std::int64_t floor_ns() const { return n_ >= 0 ? n_ / d_ : -((-n_ + d_ - 1) / d_); }

  private:
    static Rational from128(__int128 n, __int128 d) {
        if (d < 0) n = -n, d = -d;
        __int128 a = n < 0 ? -n : n, b = d;
        while (b) {
            __int128 t = a % b;
            a = b;
            b = t;
        }
        if (a > 1) n /= a, d /= a;
        if (n > INT64_MAX || n < INT64_MIN || d > INT64_MAX) throw std::overflow_error("Rational: int64 overflow");
        Rational r;
        r.n_ = (std::int64_t)n;
        r.d_ = (std::int64_t)d;
        return r;
    }
    void norm() {
        if (d_ < 0) n_ = -n_, d_ = -d_;
        std::int64_t g = std::gcd(n_ < 0 ? -n_ : n_, d_);
        if (g > 1) n_ /= g, d_ /= g;
    }
    std::int64_t n_, d_;
};
inline std::int64_t numerator(const Rational& r) { return r.num(); }
inline std::int64_t denominator(const Rational& r) { return r.den(); }

// ---------------------------------------------------------------- ids
template <class Tag>
struct Id {  // ids.hpp:11-19
    std::int32_t value = -1;
    constexpr Id() = default;
    constexpr explicit Id(std::int32_t v) : value(v) {}
    constexpr bool valid() const { return value >= 0; }
    friend constexpr bool operator==(const Id& a, const Id& b) { return a.value == b.value; }
    friend constexpr bool operator!=(const Id& a, const Id& b) { return a.value != b.value; }
    friend constexpr bool operator<(const Id& a, const Id& b) { return a.value < b.value; }
};
using VctxId = Id<struct VctxTag>;
using PctxId = Id<struct PctxTag>;
using KernelId = Id<struct KernelTag>;
using DeviceId = Id<struct DeviceTag>;
using RequestId = Id<struct RequestTag>;

// ---------------------------------------------------------------- core types
enum class Phase { Prefill, Decode, Training, Other };             // types.hpp:23
enum class PriorityClass { LatencyCritical, BestEffort };           // types.hpp:24

struct KernelSignature {  // types.hpp:29-34
    std::string semantic_id;
    std::int64_t grid_size = 1;
    friend bool operator==(const KernelSignature& a, const KernelSignature& b) {
        return a.semantic_id == b.semantic_id && a.grid_size == b.grid_size;
    }
};

struct Kernel {  // the policy-visible part of the immutable launch record (types.hpp:46-68)
    KernelId id;
    VctxId vctx;
    KernelSignature signature;
    Rational base_duration;       // ns hint (the predictor's cold start)
    Rational compute_saturation;  // s in (0, 1]
    Phase phase = Phase::Other;
    Rational arrival_floor;
    RequestId request;
    int decode_index = -1;
};

struct SloSpec {  // policy.hpp:17-22
    Rational ttft_deadline;
    Rational tpot_deadline;
    std::optional<Rational> e2e_deadline;
};

// The engine's predictor as the hooks see it (valid during a callback).
class DurationPredictor {
  public:
    explicit DurationPredictor(const void* handle = nullptr) : h_(handle) {}
    Rational predict(const KernelSignature& sig, const std::optional<Rational>& hint = std::nullopt) const {
        std::int64_t out = 0;
        check(ds_predictor_predict(h_, sig.semantic_id.c_str(), sig.grid_size, hint ? 1 : 0,
                                   hint ? hint->floor_ns() : 0, &out));
        return Rational(out);
    }
    const void* handle() const { return h_; }

  private:
    const void* h_;
};

struct PolicyView {  // policy.hpp:24-69
    struct QueuedEntry {
        KernelSignature signature;
        Rational base_hint;
    };
    struct PctxEntry {
        PctxId id;
        DeviceId device;
        Rational tier;
        bool standby = false;
        std::optional<VctxId> bound;
        bool available = true;
        std::optional<KernelId> running_kernel;
        KernelSignature running_signature;
        Rational running_remaining;
        Phase running_phase = Phase::Other;
        PriorityClass running_priority = PriorityClass::BestEffort;
        std::vector<QueuedEntry> queued;  // hw_queue depth 1: never filled
    };
    struct VctxEntry {
        VctxId id;
        PriorityClass priority = PriorityClass::BestEffort;
        bool quarantined = false;
        bool bound = false;
        std::int64_t pending = 0;
        Phase head_phase = Phase::Other;
        bool decoding = false;
    };
    Rational now;
    std::vector<PctxEntry> pctxs;
    std::vector<VctxEntry> vctxs;
    std::map<DeviceId, Rational> bound_tier_sums;
    std::map<DeviceId, Rational> min_tiers;
    const DurationPredictor* predictor = nullptr;
    std::int64_t active_vctx_count = 0;

    const PctxEntry* pctx(PctxId id) const {
        for (const auto& p : pctxs)
            if (p.id == id) return &p;
        return nullptr;
    }
    const VctxEntry* vctx(VctxId id) const {
        for (const auto& v : vctxs)
            if (v.id == id) return &v;
        return nullptr;
    }
    bool feasible_bind(const PctxEntry& p) const {
        auto it = bound_tier_sums.find(p.device);
        Rational sum = it == bound_tier_sums.end() ? Rational(0) : it->second;
        return sum + p.tier <= Rational(1);
    }
};

struct LaunchContext {  // policy.hpp:71-78
    VctxId vctx;
    const Kernel* kernel = nullptr;
    Rational request_arrival;
    std::optional<SloSpec> slo;
    bool pool_exhausted = false;
};

struct PolicyDecision {  // policy.hpp:80-90
    enum class Kind { DispatchDirect, DispatchRemap, DispatchDefer, Preempt, NoAction };
    Kind kind = Kind::NoAction;
    PctxId target;
    static PolicyDecision direct() { return {Kind::DispatchDirect, {}}; }
    static PolicyDecision remap(PctxId to) { return {Kind::DispatchRemap, to}; }
    static PolicyDecision defer() { return {Kind::DispatchDefer, {}}; }
    static PolicyDecision preempt(PctxId victim) { return {Kind::Preempt, victim}; }
    static PolicyDecision no_action() { return {Kind::NoAction, {}}; }
};

inline Rational predict_hol_blocking(const PolicyView& view, const PolicyView::PctxEntry& pctx,
                                     const DurationPredictor& predictor) {  // policy.hpp:92-95
    (void)view;
    Rational total = pctx.running_kernel ? pctx.running_remaining : Rational(0);
    for (const auto& q : pctx.queued) total += predictor.predict(q.signature, q.base_hint);
    return total;
}

class Policy {  // policy.hpp:97-126
  public:
    virtual ~Policy() = default;
    virtual std::string_view name() const = 0;
    virtual PolicyDecision on_launch(const PolicyView& view, const LaunchContext& launch) const = 0;
    virtual PolicyDecision on_completion(const PolicyView& view, const LaunchContext& next) const {
        (void)view;
        (void)next;
        return PolicyDecision::no_action();
    }
    virtual PolicyDecision on_congestion(const PolicyView& view, const LaunchContext& launch) const {
        (void)view;
        (void)launch;
        return PolicyDecision::defer();
    }
    virtual int launch_order_key(const LaunchContext& launch) const {
        (void)launch;
        return 0;
    }
    virtual std::optional<Rational> next_review_time(const PolicyView& view) const {
        (void)view;
        return std::nullopt;
    }
};

// ---------------------------------------------------------------- C <-> C++ views
namespace detail {

struct ViewHolder {  // a PolicyView plus the objects its pointers refer to
    PolicyView view;
    DurationPredictor predictor;
};

inline void from_c(const ds_view& c, ViewHolder& h) {
    PolicyView& v = h.view;
    v = PolicyView{};
    h.predictor = DurationPredictor(c.predictor);
    v.predictor = c.predictor ? &h.predictor : nullptr;
    v.now = Rational(c.now_ns);
    for (int i = 0; i < c.n_pctx; ++i) {
        const ds_view_pctx& p = c.pctx[i];
        PolicyView::PctxEntry e;
        e.id = PctxId(p.id);
        e.device = DeviceId(p.device);
        e.tier = Rational(p.tier_num, p.tier_den);
        e.standby = p.standby != 0;
        e.available = p.available != 0;
        if (p.bound >= 0) e.bound = VctxId(p.bound);
        if (p.has_running) e.running_kernel = KernelId((std::int32_t)p.running_kernel);
        e.running_signature = KernelSignature{p.running_semantic_id ? p.running_semantic_id : "", p.running_grid};
        e.running_remaining = Rational(p.running_remaining_ns);
        e.running_phase = (Phase)p.running_phase;
        e.running_priority = (PriorityClass)p.running_priority;
        v.pctxs.push_back(std::move(e));
    }
    for (int i = 0; i < c.n_vctx; ++i) {
        const ds_view_vctx& x = c.vctx[i];
        PolicyView::VctxEntry e;
        e.id = VctxId(x.id);
        e.priority = (PriorityClass)x.priority;
        e.quarantined = x.quarantined != 0;
        e.bound = x.bound != 0;
        e.pending = x.pending;
        e.head_phase = (Phase)x.head_phase;
        e.decoding = x.decoding != 0;
        v.vctxs.push_back(e);
    }
    for (int d = 0; d < c.n_devices; ++d) {
        v.bound_tier_sums[DeviceId(d)] = Rational(c.bound_tier_sum_num[d], c.bound_tier_sum_den[d]);
        v.min_tiers[DeviceId(d)] = Rational(c.min_tier_num[d], c.min_tier_den[d]);
    }
    v.active_vctx_count = c.active_vctx_count;
}

struct LaunchHolder {
    LaunchContext launch;
    Kernel kernel;
};

inline void from_c(const ds_launch_ctx& c, LaunchHolder& h) {
    h.launch = LaunchContext{};
    h.launch.vctx = VctxId(c.vctx);
    h.launch.request_arrival = Rational(c.request_arrival_ns);
    h.launch.pool_exhausted = c.pool_exhausted != 0;
    if (c.has_slo) h.launch.slo = SloSpec{Rational(c.ttft_ns), Rational(c.tpot_ns), std::nullopt};
    if (c.has_kernel) {
        Kernel& k = h.kernel;
        k = Kernel{};
        k.id = KernelId((std::int32_t)c.kernel_id);
        k.vctx = VctxId(c.vctx);
        k.signature = KernelSignature{c.semantic_id ? c.semantic_id : "", c.grid_size};
        k.base_duration = Rational(c.base_hint_ns);
        k.compute_saturation = Rational(c.sat_num, c.sat_den);
        k.phase = (Phase)c.phase;
        k.arrival_floor = Rational(c.arrival_ns);
        k.request = RequestId((std::int32_t)c.request);
        k.decode_index = c.decode_index;
        h.launch.kernel = &k;
    }
}

inline ds_decision to_c(const PolicyDecision& d) { return ds_decision{(std::int32_t)d.kind, d.target.value}; }

// vtable trampolines: user = the Policy object (owned by the engine)
inline ds_decision decide(int which, void* user, const ds_view* v, const ds_launch_ctx* l) {
    const Policy* p = static_cast<const Policy*>(user);
    ViewHolder vh;
    from_c(*v, vh);
    LaunchHolder lh;
    from_c(*l, lh);
    try {
        switch (which) {
            case 0: return to_c(p->on_launch(vh.view, lh.launch));
            case 1: return to_c(p->on_completion(vh.view, lh.launch));
            default: return to_c(p->on_congestion(vh.view, lh.launch));
        }
    } catch (...) {  // no exceptions across the C ABI: an out-of-range value is an illegal decision
        return ds_decision{-1, -1};
    }
}
inline void on_launch_tr(void* u, const ds_view* v, const ds_launch_ctx* l, ds_decision* o) { *o = decide(0, u, v, l); }
inline void on_completion_tr(void* u, const ds_view* v, const ds_launch_ctx* l, ds_decision* o) {
    *o = decide(1, u, v, l);
}
inline void on_congestion_tr(void* u, const ds_view* v, const ds_launch_ctx* l, ds_decision* o) {
    *o = decide(2, u, v, l);
}
inline int order_key_tr(void* u, const ds_launch_ctx* l) {
    LaunchHolder lh;
    from_c(*l, lh);
    return static_cast<const Policy*>(u)->launch_order_key(lh.launch);
}
inline int review_tr(void* u, const ds_view* v, std::int64_t* t) {
    ViewHolder vh;
    from_c(*v, vh);
    auto r = static_cast<const Policy*>(u)->next_review_time(vh.view);
    if (!r) return 0;
    *t = r->floor_ns();
    return 1;
}
inline void destroy_tr(void* u) { delete static_cast<Policy*>(u); }

}  // namespace detail

// ---------------------------------------------------------------- built-in policies
struct PolicyConfig {  // policies.hpp:12-18 (times in ns)
    std::string name = "slo-aware";
    Rational quantum{5000000};
    Rational predictor_alpha{3, 10};
    Rational cold_start_prediction{1000000000};
    std::map<VctxId, PctxId> assignments;
};

// A built-in policy: its hooks are the native implementation's
// (ds_builtin_decide); an engine given one runs it natively.
class BuiltinPolicy : public Policy {
  public:
    explicit BuiltinPolicy(PolicyConfig cfg) : cfg_(std::move(cfg)) {}
    std::string_view name() const override { return cfg_.name; }
    PolicyDecision on_launch(const PolicyView& v, const LaunchContext& l) const override { return decide(0, v, l); }
    PolicyDecision on_completion(const PolicyView& v, const LaunchContext& l) const override { return decide(1, v, l); }
    PolicyDecision on_congestion(const PolicyView& v, const LaunchContext& l) const override { return decide(2, v, l); }
    int launch_order_key(const LaunchContext& l) const override { return decide(3, PolicyView{}, l).target.value; }
    std::optional<Rational> next_review_time(const PolicyView& v) const override {  // policies.cpp:256-258
        if (cfg_.name != "temporal") return std::nullopt;
        std::int64_t q = cfg_.quantum.floor_ns();
        return Rational((v.now.floor_ns() / q + 1) * q);
    }
    const PolicyConfig& config() const { return cfg_; }

  private:
    PolicyDecision decide(int hook, const PolicyView& v, const LaunchContext& l) const;
    PolicyConfig cfg_;
};

struct SloAwarePolicy : BuiltinPolicy {
    SloAwarePolicy() : BuiltinPolicy(PolicyConfig{"slo-aware"}) {}
};
struct TpotFirstPolicy : BuiltinPolicy {
    TpotFirstPolicy() : BuiltinPolicy(PolicyConfig{"tpot-first"}) {}
};
struct TemporalBaselinePolicy : BuiltinPolicy {
    explicit TemporalBaselinePolicy(Rational quantum) : BuiltinPolicy(PolicyConfig{"temporal", quantum}) {}
};

inline std::unique_ptr<Policy> make_policy(const PolicyConfig& config) {  // policies.hpp:74
    char names[256];
    check_engine(ds_policy_names(names, sizeof names));
    std::string all = std::string(",") + names + ",";
    if (all.find("," + config.name + ",") == std::string::npos)
        throw SimError(DS_CONFIG_ERROR, "unknown policy '" + config.name + "' (valid: " + names + ")");
    return std::make_unique<BuiltinPolicy>(config);
}

inline std::vector<std::string> policy_names() {  // policies.hpp:75
    char names[256];
    check_engine(ds_policy_names(names, sizeof names));
    std::vector<std::string> out;
    std::string s = names;
    for (std::size_t a = 0, b; a <= s.size(); a = b + 1) {
        b = s.find(',', a);
        if (b == std::string::npos) b = s.size();
        if (b > a) out.push_back(s.substr(a, b - a));
    }
    return out;
}

namespace detail {
inline void to_c(const PolicyView& v, ds_view& c, std::vector<std::string>& keep) {
    std::memset(&c, 0, sizeof c);
    c.now_ns = v.now.floor_ns();
    c.n_pctx = (int)std::min<std::size_t>(v.pctxs.size(), DS_VIEW_MAX_PCTX);
    keep.reserve(c.n_pctx);
    for (int i = 0; i < c.n_pctx; ++i) {
        const auto& p = v.pctxs[i];
        ds_view_pctx& o = c.pctx[i];
        o.id = p.id.value;
        o.device = p.device.value < 0 ? 0 : p.device.value;
        o.tier_num = p.tier.num();
        o.tier_den = p.tier.den();
        o.standby = p.standby;
        o.available = p.available;
        o.bound = p.bound ? p.bound->value : -1;
        o.has_running = p.running_kernel.has_value();
        o.running_kernel = p.running_kernel ? (std::uint64_t)p.running_kernel->value : 0;
        keep.push_back(p.running_signature.semantic_id);
        o.running_semantic_id = keep.back().c_str();
        o.running_grid = p.running_signature.grid_size;
        o.running_remaining_ns = p.running_remaining.floor_ns();
        o.running_phase = (int)p.running_phase;
        o.running_priority = (int)p.running_priority;
    }
    c.n_vctx = (int)std::min<std::size_t>(v.vctxs.size(), DS_VIEW_MAX_VCTX);
    for (int i = 0; i < c.n_vctx; ++i) {
        const auto& x = v.vctxs[i];
        ds_view_vctx& o = c.vctx[i];
        o.id = x.id.value;
        o.priority = (int)x.priority;
        o.quarantined = x.quarantined;
        o.bound = x.bound;
        o.pending = x.pending;
        o.head_phase = (int)x.head_phase;
        o.decoding = x.decoding;
    }
    int nd = 0;
    for (const auto& kv : v.bound_tier_sums) nd = std::max(nd, kv.first.value + 1);
    for (const auto& kv : v.min_tiers) nd = std::max(nd, kv.first.value + 1);
    c.n_devices = std::min(nd, DS_VIEW_MAX_DEVICES);
    for (int d = 0; d < c.n_devices; ++d) {
        auto b = v.bound_tier_sums.find(DeviceId(d));
        auto m = v.min_tiers.find(DeviceId(d));
        Rational bs = b == v.bound_tier_sums.end() ? Rational(0) : b->second;
        Rational mt = m == v.min_tiers.end() ? Rational(1) : m->second;
        c.bound_tier_sum_num[d] = bs.num();
        c.bound_tier_sum_den[d] = bs.den();
        c.min_tier_num[d] = mt.num();
        c.min_tier_den[d] = mt.den();
    }
    c.active_vctx_count = v.active_vctx_count;
    c.predictor = v.predictor ? v.predictor->handle() : nullptr;
}

inline void to_c(const LaunchContext& l, ds_launch_ctx& c) {
    std::memset(&c, 0, sizeof c);
    c.vctx = l.vctx.value;
    c.request_arrival_ns = l.request_arrival.floor_ns();
    c.pool_exhausted = l.pool_exhausted;
    c.request = -1;
    c.decode_index = -1;
    c.phase = (int)Phase::Other;
    c.sat_num = c.sat_den = 1;
    if (l.slo) {
        c.has_slo = 1;
        c.ttft_ns = l.slo->ttft_deadline.floor_ns();
        c.tpot_ns = l.slo->tpot_deadline.floor_ns();
    }
    if (l.kernel) {
        const Kernel& k = *l.kernel;
        c.has_kernel = 1;
        c.kernel_id = (std::uint64_t)k.id.value;
        c.semantic_id = k.signature.semantic_id.c_str();
        c.grid_size = k.signature.grid_size;
        c.base_hint_ns = k.base_duration.floor_ns();
        c.sat_num = k.compute_saturation.num();
        c.sat_den = k.compute_saturation.den();
        c.phase = (int)k.phase;
        c.decode_index = k.decode_index;
        c.request = k.request.value;
        c.arrival_ns = k.arrival_floor.floor_ns();
    }
}
}  // namespace detail

inline PolicyDecision BuiltinPolicy::decide(int hook, const PolicyView& v, const LaunchContext& l) const {
    auto cv = std::make_unique<ds_view>();
    std::vector<std::string> keep;
    detail::to_c(v, *cv, keep);
    ds_launch_ctx cl;
    detail::to_c(l, cl);
    ds_decision d{};
    check_engine(ds_builtin_decide(cfg_.name.c_str(), hook, cv.get(), &cl, cfg_.quantum.floor_ns(), &d));
    return PolicyDecision{(PolicyDecision::Kind)d.kind, PctxId(d.target)};
}

// ---------------------------------------------------------------- device / pool
// create_pool (types.hpp:133-137) over one GPU sharing domain: one pctx per
// tier, floor(tier x #SMs) SMs each.  Tenants (the reference's jobs/vctxs)
// and their device kernels (immutable launch records) are registered here.
class Device {
  public:
    Device(int cuda_device, const std::vector<Rational>& tiers, int block_log_capacity = 0, bool lend_idle_sms = true) {
        ds_domain_config cfg;
        std::memset(&cfg, 0, sizeof cfg);
        cfg.device = cuda_device;
        cfg.n_tiers = (int)tiers.size();
        if (tiers.empty() || tiers.size() > 16) throw SimError(DS_INVALID_TIER, "pool needs 1..16 tiers");
        for (std::size_t i = 0; i < tiers.size(); ++i) {
            cfg.tier_num[i] = tiers[i].num();
            cfg.tier_den[i] = tiers[i].den();
        }
        cfg.block_log_capacity = block_log_capacity;
        cfg.lend_idle_sms = lend_idle_sms ? 1 : 0;
        check(ds_domain_create(&cfg, &h_));
    }
    ~Device() {
        if (h_) {
            ds_stop(h_);
            ds_domain_destroy(h_);
        }
    }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;

    ds_domain* handle() const { return h_; }
    int num_sms() const {
        int n = 0;
        check(ds_num_sms(h_, &n));
        return n;
    }
    int pctx_count() const {
        int n = 0;
        check(ds_pctx_count(h_, &n));
        return n;
    }
    VctxId add_tenant(const std::string& name, PriorityClass p) {
        ds_tenant_desc d{name.c_str(), (int)p};
        int id = -1;
        check(ds_tenant_register(h_, &d, &id));
        return VctxId(id);
    }
    // an immutable device kernel (body + logical grid + argument block)
    int add_kernel(const std::string& semantic_id, int body, std::uint32_t gx, std::uint32_t gy, std::uint32_t gz,
                   const void* args, std::uint32_t args_size, Phase phase = Phase::Other) {
        ds_kernel_desc k;
        std::memset(&k, 0, sizeof k);
        k.semantic_id = semantic_id.c_str();
        k.body = body;
        k.grid_x = gx;
        k.grid_y = gy;
        k.grid_z = gz;
        k.block_threads = 256;
        k.args = args;
        k.args_size = args_size;
        k.phase = (int)phase;
        k.request = -1;
        k.decode_index = -1;
        int id = -1;
        check(ds_kernel_register(h_, &k, &id));
        return id;
    }
    void start() { check(ds_start(h_)); }
    void stop() { check(ds_stop(h_)); }

  private:
    ds_domain* h_ = nullptr;
};

inline std::unique_ptr<Device> create_pool(int cuda_device, const std::vector<Rational>& tiers) {
    return std::make_unique<Device>(cuda_device, tiers);
}
inline void bind(Device& d, VctxId v, PctxId p) { check(ds_bind(d.handle(), v.value, p.value)); }  // types.cpp:62-74
inline void unbind(Device& d, VctxId v) { check(ds_unbind(d.handle(), v.value)); }                // types.cpp:76-85

// exclusive_baseline (engine.cpp:1400-1417): the same kernel alone, as a
// plain grid on the whole GPU (stream: a cudaStream_t, or nullptr)
inline void exclusive_baseline(Device& d, int kernel, void* stream = nullptr) {
    check(ds_solo_launch_registered(d.handle(), kernel, stream));
}

// ---------------------------------------------------------------- engine
struct EngineConfig {  // engine.hpp:58-72 (the parts that apply to real hardware)
    bool release_on_idle = true;
    bool hang_detection = false;
    Rational hang_threshold{3};
    Rational reset_delay{200000};  // ns
    bool capture_log = false;
    bool fair_handover = true;     // temporal: hand the device over at each quantum
    int lend_tenant = -1;          // tenant run on unbound SMs (-1: idle SMs stay idle)
};

struct RecordSpec {  // one Kernel launch record: >= 1 device kernels in program order
    std::string semantic_id;
    std::int64_t grid_size = 1;
    std::vector<int> kernels;
    Phase phase = Phase::Other;
    std::int64_t request = -1;
    int decode_index = -1;
    std::optional<SloSpec> slo;
    Rational base_hint;
    Rational compute_saturation{1};
    Rational arrival;           // engine ns; 0 = now
    Rational request_arrival;   // engine ns; 0 = arrival
};

struct EngineCounters {
    std::uint64_t decisions = 0, dispatches = 0, completed = 0, preemptions = 0, migrations = 0, unbinds = 0,
                  policy_errors = 0, failed_jobs = 0;
};

// SimEngine (engine.hpp:152-170) over a Device: the same dispatch loop
// (pump_launches / apply_decision / preempt at block boundaries / migrate)
// driving the executor.  With a user Policy the engine owns it.
class SimEngine {
  public:
    explicit SimEngine(Device& dev, EngineConfig config = {}, std::unique_ptr<Policy> policy = nullptr,
                       PolicyConfig pconf = {}) {
        ds_engine_config cfg;
        std::memset(&cfg, 0, sizeof cfg);
        cfg.release_on_idle = config.release_on_idle;
        cfg.hang_detection = config.hang_detection;
        cfg.hang_threshold = (double)config.hang_threshold.num() / (double)config.hang_threshold.den();
        cfg.reset_delay_ns = config.reset_delay.floor_ns();
        cfg.capture_log = config.capture_log;
        cfg.fair_handover = config.fair_handover;
        cfg.lend_tenant = config.lend_tenant;
        cfg.alpha = (double)pconf.predictor_alpha.num() / (double)pconf.predictor_alpha.den();
        cfg.cold_start_ns = pconf.cold_start_prediction.floor_ns();
        cfg.quantum_ns = pconf.quantum.floor_ns();
        int i = 0;
        for (const auto& kv : pconf.assignments) {
            if (i >= 64) break;
            cfg.assign_vctx[i] = kv.first.value;
            cfg.assign_pctx[i] = kv.second.value;
            ++i;
        }
        cfg.n_assignments = i;
        auto* builtin = dynamic_cast<BuiltinPolicy*>(policy.get());
        if (!policy || builtin) {  // built-in: runs natively
            std::string name = builtin ? builtin->config().name : pconf.name;
            if (builtin) cfg.quantum_ns = builtin->config().quantum.floor_ns();
            cfg.policy = name.c_str();
            check_engine(ds_engine_create(dev.handle(), &cfg, &h_));
            return;
        }
        name_ = std::string(policy->name());
        ds_policy_vtable vt;
        vt.name = name_.c_str();
        vt.on_launch = detail::on_launch_tr;
        vt.on_completion = detail::on_completion_tr;
        vt.on_congestion = detail::on_congestion_tr;
        vt.launch_order_key = detail::order_key_tr;
        vt.next_review_time = detail::review_tr;
        vt.destroy = detail::destroy_tr;
        Policy* raw = policy.release();
        int st = ds_engine_create_with_policy(dev.handle(), &cfg, &vt, raw, &h_);
        if (st) {
            delete raw;
            check_engine(st);
        }
    }
    ~SimEngine() {
        if (h_) ds_engine_destroy(h_);
    }
    SimEngine(const SimEngine&) = delete;
    SimEngine& operator=(const SimEngine&) = delete;

    int add_job(VctxId tenant, PriorityClass p) {
        int j = -1;
        check_engine(ds_engine_add_job(h_, tenant.value, (int)p, &j));
        return j;
    }
    KernelId submit(int job, const RecordSpec& r) {
        ds_record_desc d;
        std::memset(&d, 0, sizeof d);
        d.semantic_id = r.semantic_id.c_str();
        d.grid_size = r.grid_size;
        d.kernels = r.kernels.data();
        d.n_kernels = (int)r.kernels.size();
        d.phase = (int)r.phase;
        d.request = r.request;
        d.decode_index = r.decode_index;
        d.arrival_ns = r.arrival.floor_ns();
        d.request_arrival_ns = r.request_arrival.floor_ns();
        if (r.slo) {
            d.ttft_ns = r.slo->ttft_deadline.floor_ns();
            d.tpot_ns = r.slo->tpot_deadline.floor_ns();
        }
        d.base_hint_ns = r.base_hint.floor_ns();
        d.sat_num = r.compute_saturation.num();
        d.sat_den = r.compute_saturation.den();
        std::uint64_t id = 0;
        check_engine(ds_engine_submit(h_, job, &d, &id));
        return KernelId((std::int32_t)id);
    }
    void start() { check_engine(ds_engine_start(h_)); }
    void stop() { check_engine(ds_engine_stop(h_)); }
    void wait(KernelId k, int timeout_ms = 60000) { check_engine(ds_engine_wait(h_, (std::uint64_t)k.value, timeout_ms)); }
    EngineCounters counters() const {
        ds_engine_counters c;
        check_engine(ds_engine_counters_get(h_, &c));
        return EngineCounters{c.decisions, c.dispatches, c.completed, c.preemptions, c.migrations, c.unbinds,
                              c.policy_errors, c.failed_jobs};
    }
    // ds_snapshot: the PolicyView a hook would see now (no predictor pointer)
    PolicyView snapshot() const {
        auto c = std::make_unique<ds_view>();
        check_engine(ds_engine_snapshot(h_, c.get()));
        detail::ViewHolder vh;
        detail::from_c(*c, vh);
        vh.view.predictor = nullptr;
        return vh.view;
    }
    ds_engine* handle() const { return h_; }

  private:
    ds_engine* h_ = nullptr;
    std::string name_;
};

}  // namespace corosim
