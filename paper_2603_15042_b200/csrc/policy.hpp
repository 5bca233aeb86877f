// Scheduling policy API of the B200 runtime — the reference's Policy surface
// (proj/include/corosim/policy/policy.hpp:17-126, policies.hpp:12-75,
// predictor.hpp:14-31) with the same hooks, names and decision semantics,
// over real device state.  Time is integer nanoseconds (host steady clock for
// decisions, %globaltimer for measured durations); tiers are exact fractions.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "../../include/detshare/ds.h"

namespace detshare {

using Time = int64_t;  // ns

struct Frac {  // exact tier fraction (QuotaTier, types.hpp:19-21)
    int64_t num = 0, den = 1;
    friend bool operator<(const Frac& a, const Frac& b) { return (__int128)a.num * b.den < (__int128)b.num * a.den; }
    friend bool operator==(const Frac& a, const Frac& b) { return (__int128)a.num * b.den == (__int128)b.num * a.den; }
    friend bool operator!=(const Frac& a, const Frac& b) { return !(a == b); }
    friend bool operator<=(const Frac& a, const Frac& b) { return !(b < a); }
    friend bool operator>(const Frac& a, const Frac& b) { return b < a; }
    friend bool operator>=(const Frac& a, const Frac& b) { return !(a < b); }
    friend Frac operator+(const Frac& a, const Frac& b);
    double value() const { return (double)num / (double)den; }
};

enum class Phase { Prefill, Decode, Training, Other };          // types.hpp:23
enum class PriorityClass { LatencyCritical, BestEffort };        // types.hpp:24

struct KernelSignature {  // types.hpp:29-34
    std::string semantic_id;
    int64_t grid_size = 1;
    bool operator==(const KernelSignature& o) const { return semantic_id == o.semantic_id && grid_size == o.grid_size; }
};

struct SloSpec {  // policy.hpp:17-22
    Time ttft_deadline = 0;
    Time tpot_deadline = 0;
};

// A launch record as the policy sees it (the reference's Kernel record,
// types.hpp:46-68): one policy unit, executed as >= 1 device kernels.
struct LaunchRecord {
    uint64_t id = 0;
    int job = -1;
    KernelSignature signature;
    Time base_duration = 0;        // hint for the predictor (ns)
    Frac compute_saturation{1, 1};
    Phase phase = Phase::Other;
    int64_t request = -1;
    int decode_index = -1;
    std::optional<SloSpec> slo;
    Time arrival = 0;              // host ns (engine clock)
    Time request_arrival = 0;
    std::vector<int32_t> kernels;  // registered device kernel ids, program order
};

class DurationPredictor {  // predictor.hpp:14-31, predictor.cpp:7-38
  public:
    explicit DurationPredictor(double alpha = 0.3, Time cold_default = 1000000000);
    void observe(const KernelSignature& sig, Time effective_duration);
    Time predict(const KernelSignature& sig, std::optional<Time> hint = std::nullopt) const;
    bool has_observation(const KernelSignature& sig) const;

  private:
    double alpha_;
    Time cold_default_;
    std::map<std::pair<std::string, int64_t>, double> ewma_;
    std::map<std::string, Time> max_by_semantic_;
};

struct PolicyView {  // policy.hpp:24-69
    struct QueuedEntry {
        KernelSignature signature;
        Time base_hint = 0;
    };
    struct PctxEntry {
        int id = -1;
        int device = 0;
        Frac tier;
        bool standby = false;
        std::optional<int> bound;
        bool available = true;
        std::optional<uint64_t> running_kernel;
        KernelSignature running_signature;
        Time running_remaining = 0;
        Phase running_phase = Phase::Other;
        PriorityClass running_priority = PriorityClass::BestEffort;
        std::vector<QueuedEntry> queued;
    };
    struct VctxEntry {
        int id = -1;
        PriorityClass priority = PriorityClass::BestEffort;
        bool quarantined = false;
        bool bound = false;
        int64_t pending = 0;
        Phase head_phase = Phase::Other;
        bool decoding = false;
    };
    Time now = 0;
    std::vector<PctxEntry> pctxs;
    std::vector<VctxEntry> vctxs;
    std::map<int, Frac> bound_tier_sums;
    std::map<int, Frac> min_tiers;
    const DurationPredictor* predictor = nullptr;
    int64_t active_vctx_count = 0;

    const PctxEntry* pctx(int id) const;
    const VctxEntry* vctx(int id) const;
    bool feasible_bind(const PctxEntry& p) const;
};

struct LaunchContext {  // policy.hpp:71-78
    int vctx = -1;
    const LaunchRecord* kernel = nullptr;
    Time request_arrival = 0;
    std::optional<SloSpec> slo;
    bool pool_exhausted = false;
};

struct PolicyDecision {  // policy.hpp:80-90
    enum class Kind { DispatchDirect, DispatchRemap, DispatchDefer, Preempt, NoAction };
    Kind kind = Kind::NoAction;
    int target = -1;
    static PolicyDecision direct() { return {Kind::DispatchDirect, -1}; }
    static PolicyDecision remap(int to) { return {Kind::DispatchRemap, to}; }
    static PolicyDecision defer() { return {Kind::DispatchDefer, -1}; }
    static PolicyDecision preempt(int victim) { return {Kind::Preempt, victim}; }
    static PolicyDecision no_action() { return {Kind::NoAction, -1}; }
};

Time predict_hol_blocking(const PolicyView& view, const PolicyView::PctxEntry& pctx, const DurationPredictor& predictor);

class Policy {  // policy.hpp:97-126
  public:
    virtual ~Policy() = default;
    virtual std::string_view name() const = 0;
    virtual PolicyDecision on_launch(const PolicyView& view, const LaunchContext& launch) const = 0;
    virtual PolicyDecision on_completion(const PolicyView&, const LaunchContext&) const {
        return PolicyDecision::no_action();
    }
    virtual PolicyDecision on_congestion(const PolicyView&, const LaunchContext&) const {
        return PolicyDecision::defer();
    }
    virtual int launch_order_key(const LaunchContext&) const { return 0; }
    virtual std::optional<Time> next_review_time(const PolicyView&) const { return std::nullopt; }
};

struct PolicyConfig {  // policies.hpp:12-18
    std::string name = "slo-aware";
    Time quantum = 5000000;  // temporal baseline slice (5 ms)
    double predictor_alpha = 0.3;
    Time cold_start_prediction = 1000000000;
    std::map<int, int> assignments;  // static partition vctx -> pctx
};

class SloAwarePolicy : public Policy {
  public:
    std::string_view name() const override { return "slo-aware"; }
    PolicyDecision on_launch(const PolicyView& view, const LaunchContext& launch) const override;
    PolicyDecision on_congestion(const PolicyView& view, const LaunchContext& launch) const override;
    int launch_order_key(const LaunchContext& launch) const override;
};

class TpotFirstPolicy : public SloAwarePolicy {
  public:
    std::string_view name() const override { return "tpot-first"; }
    PolicyDecision on_launch(const PolicyView& view, const LaunchContext& launch) const override;
    PolicyDecision on_congestion(const PolicyView& view, const LaunchContext& launch) const override;
    int launch_order_key(const LaunchContext& launch) const override;
};

class TemporalBaselinePolicy : public Policy {
  public:
    explicit TemporalBaselinePolicy(Time quantum);
    std::string_view name() const override { return "temporal"; }
    PolicyDecision on_launch(const PolicyView& view, const LaunchContext& launch) const override;
    std::optional<Time> next_review_time(const PolicyView& view) const override;
    std::optional<int> owner_at(const PolicyView& view) const;
    Time quantum() const { return quantum_; }

  private:
    Time quantum_;
};

class StaticPartitionPolicy : public Policy {
  public:
    explicit StaticPartitionPolicy(std::map<int, int> assignments);
    std::string_view name() const override { return "static"; }
    PolicyDecision on_launch(const PolicyView& view, const LaunchContext& launch) const override;

  private:
    std::map<int, int> assignments_;
};

std::unique_ptr<Policy> make_policy(const PolicyConfig& config);  // throws std::invalid_argument
const std::vector<std::string>& policy_names();

// C-ABI policies (policy_abi.cpp): a ds_policy_vtable as a Policy, and the
// PolicyView / LaunchContext <-> C snapshot conversions
std::unique_ptr<Policy> make_abi_policy(const ds_policy_vtable& vt, void* user);
void view_to_c(const PolicyView& v, ds_view* out);
void view_from_c(const ds_view& c, PolicyView& out, const DurationPredictor* fallback);
void launch_from_c(const ds_launch_ctx& c, LaunchRecord& rec_storage, LaunchContext& out);

}  // namespace detshare
