// Request metrics over measured outcomes — the reference's compute_metrics
// (proj/src/io/metrics.cpp:9-85) on integer-ns device timestamps.  TTFT
// samples are integers; TPOT samples are exact ratios (span / (tokens - 1)),
// ordered by cross-multiplication, so percentiles and SLO violations match
// the reference's exact rationals; means and rates are reported as doubles.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

#include "../../include/detshare/ds.h"

namespace {

struct Ratio {
    int64_t num, den;  // den > 0
};
bool less(const Ratio& a, const Ratio& b) { return (__int128)a.num * b.den < (__int128)b.num * a.den; }

Ratio reduce(Ratio r) {
    int64_t g = std::gcd(r.num < 0 ? -r.num : r.num, r.den);
    if (g > 1) {
        r.num /= g;
        r.den /= g;
    }
    return r;
}

// nearest_rank_percentile (metrics.cpp:9-16): k = ceil(pct n / 100), >= 1
Ratio nearest_rank(const std::vector<Ratio>& sorted, int pct) {
    size_t n = sorted.size();
    size_t k = ((size_t)pct * n + 99) / 100;
    if (k == 0) k = 1;
    return reduce(sorted[k - 1]);
}

void summarize(std::vector<Ratio> s, ds_dist* d) {
    *d = ds_dist{};
    d->count = (int64_t)s.size();
    if (s.empty()) return;
    std::sort(s.begin(), s.end(), less);
    long double sum = 0;
    for (const Ratio& x : s) sum += (long double)x.num / (long double)x.den;
    d->mean = (double)(sum / (long double)s.size());
    Ratio p50 = nearest_rank(s, 50), p90 = nearest_rank(s, 90), p99 = nearest_rank(s, 99);
    d->p50_num = p50.num;
    d->p50_den = p50.den;
    d->p90_num = p90.num;
    d->p90_den = p90.den;
    d->p99_num = p99.num;
    d->p99_den = p99.den;
}

}  // namespace

extern "C" int ds_compute_metrics(const ds_request_outcome* reqs, int64_t n, int64_t makespan_ns,
                                  int64_t kernels_completed, ds_metrics* out) {
    if (!out || (n > 0 && !reqs) || n < 0) return DS_INVALID_ARGUMENT;
    ds_metrics m{};
    m.makespan_ns = makespan_ns;
    m.kernels_completed = kernels_completed;
    std::vector<Ratio> ttft, tpot;
    for (int64_t i = 0; i < n; ++i) {
        const ds_request_outcome& r = reqs[i];
        if (!r.inference || !r.completed) continue;
        m.inference_completed++;
        const int64_t t = r.first_decode_finish_ns - r.arrival_ns;
        ttft.push_back({t, 1});
        bool has_tpot = false;
        Ratio tp{0, 1};
        if (r.output_tokens >= 2) {
            tp = {r.last_finish_ns - r.first_decode_finish_ns, (int64_t)r.output_tokens - 1};
            tpot.push_back(tp);
            has_tpot = true;
        } else {
            m.tpot_excluded++;
        }
        if (r.has_slo) {
            m.slo_requests++;
            if (t > r.ttft_slo_ns) m.ttft_violations++;
            if (has_tpot && less(Ratio{r.tpot_slo_ns, 1}, tp)) m.tpot_violations++;
        }
    }
    summarize(ttft, &m.ttft);
    summarize(tpot, &m.tpot);
    if (m.slo_requests > 0) {
        m.ttft_violation_rate = (double)m.ttft_violations / (double)m.slo_requests;
        m.tpot_violation_rate = (double)m.tpot_violations / (double)m.slo_requests;
    }
    for (int64_t i = 0; i < n; ++i)
        if (!reqs[i].inference && reqs[i].kernels_done > 0) m.training_kernels_completed += reqs[i].kernels_done;
    if (makespan_ns > 0) {
        m.inference_throughput = (double)m.inference_completed / (double)makespan_ns;
        m.training_throughput = (double)m.training_kernels_completed / (double)makespan_ns;
    }
    *out = m;
    return DS_OK;
}

extern "C" {

// add_normalization (metrics.cpp:81-102): per job, normalized throughput =
// exclusive span / shared span (first arrival -> last finish of the job's
// kernels), 0 when either span is missing or the shared span is empty; the
// aggregate is their sum.  Exact ratios (reduced) plus doubles.
int ds_add_normalization(const ds_job_span* shared, const ds_job_span* solo, int n, int64_t* num, int64_t* den,
                         double* aggregate) {
    if ((n > 0 && (!shared || !solo || !num || !den)) || n < 0) return DS_INVALID_ARGUMENT;
    double agg = 0.0;
    for (int i = 0; i < n; ++i) {
        num[i] = 0;
        den[i] = 1;
        if (!shared[i].valid || !solo[i].valid) continue;
        const int64_t sh = shared[i].last_finish_ns - shared[i].first_arrival_ns;
        const int64_t so = solo[i].last_finish_ns - solo[i].first_arrival_ns;
        if (sh <= 0) continue;
        Ratio r = reduce(Ratio{so, sh});
        num[i] = r.num;
        den[i] = r.den;
        agg += (double)r.num / (double)r.den;
    }
    if (aggregate) *aggregate = agg;
    return DS_OK;
}

}  // extern "C"
