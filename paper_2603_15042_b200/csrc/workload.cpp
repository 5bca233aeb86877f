// Request-stream generation and workload expansion.
//
// Same arrival streams as the reference's generators, so the GPU runtime and
// the CPU simulator can be driven by identical bursty/Poisson request traces:
//   gen_poisson / gen_burst   proj/src/io/trace.cpp:189-232
//   stamp (job round-robin, token draws)   trace.cpp:164-185
//   quantize (1e-9 of the trace time unit)  trace.cpp:159-162
//   Rng (mt19937_64 + explicit transforms)  proj/include/corosim/rng.hpp:11-40
//   expand_workload (request -> kernel records, mix_seed)  proj/src/io/workload.cpp:10-16,51-174
//
// Arrival times are returned as the integer round(t * 1e9) — exactly the
// numerator of the reference's quantised Rational over 10^9 — so the two
// agree bit for bit (tests/test_workload.py pins this against the reference
// library built in oracle/_ref).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <random>
#include <vector>

#include "../../include/detshare/ds.h"

namespace {

// rng.hpp:11-40, transform for transform
class Rng {
  public:
    explicit Rng(uint64_t seed) : gen_(seed) {}
    double uniform01() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
    int64_t uniform_int(int64_t lo, int64_t hi) {
        uint64_t span = static_cast<uint64_t>(hi - lo) + 1;
        return lo + static_cast<int64_t>(gen_() % span);
    }
    double exponential(double rate) {
        double u;
        do {
            u = uniform01();
        } while (u == 0.0);
        return -std::log(u) / rate;
    }

  private:
    std::mt19937_64 gen_;
};

int64_t quantize(double t) { return static_cast<int64_t>(std::round(t * 1e9)); }

ds_request stamp(const ds_request_template& tm, Rng& rng, int index, int64_t at) {
    ds_request r{};
    r.arrival_q = at;
    r.stream = index % (tm.streams > 1 ? tm.streams : 1);
    r.kind = tm.kind;
    if (tm.kind == DS_REQ_INFERENCE) {
        // draw order: prompt, then output (trace.cpp:173-180)
        r.prompt_tokens = tm.prompt_tokens_max > tm.prompt_tokens
                              ? static_cast<int32_t>(rng.uniform_int(tm.prompt_tokens, tm.prompt_tokens_max))
                              : tm.prompt_tokens;
        r.output_tokens = tm.output_tokens_max > tm.output_tokens
                              ? static_cast<int32_t>(rng.uniform_int(tm.output_tokens, tm.output_tokens_max))
                              : tm.output_tokens;
    } else {
        r.iterations = tm.iterations;
    }
    return r;
}

struct Sink {
    ds_request* out;
    int64_t cap;
    int64_t n = 0;
    void push(const ds_request& r) {
        if (n < cap && out) out[n] = r;
        ++n;
    }
};

bool valid_template(const ds_request_template* t) {
    return t && (t->kind == DS_REQ_INFERENCE || t->kind == DS_REQ_TRAINING);
}

// workload.cpp:10-16
uint64_t mix_seed(uint64_t a, uint64_t b) {
    uint64_t h = a * 0x9e3779b97f4a7c15ULL + b + 0x517cc1b727220a95ULL;
    h ^= h >> 31;
    h *= 0xbf58476d1ce4e5b9ULL;
    h ^= h >> 29;
    return h;
}

}  // namespace

extern "C" {

int ds_gen_poisson(double rate, double duration, const ds_request_template* tmpl, uint64_t seed, ds_request* out,
                   int64_t cap, int64_t* n) {
    if (!valid_template(tmpl) || !n || cap < 0) return DS_INVALID_ARGUMENT;
    Sink s{out, cap};
    if (rate > 0 && duration > 0) {
        Rng rng(seed);
        double t = 0;
        int index = 0;
        for (;;) {
            t += rng.exponential(rate);
            if (t >= duration) break;
            s.push(stamp(*tmpl, rng, index++, quantize(t)));
        }
    }
    *n = s.n;
    return DS_OK;
}

int ds_gen_burst(double base_rate, double burst_rate, double burst_duration, double period, double duration,
                 const ds_request_template* tmpl, uint64_t seed, ds_request* out, int64_t cap, int64_t* n) {
    if (!valid_template(tmpl) || !n || cap < 0) return DS_INVALID_ARGUMENT;
    Sink s{out, cap};
    if (!(duration <= 0 || period <= 0 || burst_duration < 0 || burst_duration > period)) {
        Rng rng(seed);
        double t = 0;
        int index = 0;
        while (t < duration) {
            const double in_period = std::fmod(t, period);
            const bool bursting = in_period < burst_duration;
            const double rate = bursting ? burst_rate : base_rate;
            const double seg_end = t - in_period + (bursting ? burst_duration : period);
            if (rate <= 0) {
                t = seg_end;
                continue;
            }
            const double gap = rng.exponential(rate);
            if (t + gap >= seg_end) {  // no arrival before the rate changes
                t = seg_end;
                continue;
            }
            t += gap;
            if (t >= duration) break;
            s.push(stamp(*tmpl, rng, index++, quantize(t)));
        }
    }
    *n = s.n;
    return DS_OK;
}

// expand_workload (workload.cpp:51-174): requests in trace order; job index
// = first appearance of the stream; per request a prefill record (grid
// ceil(prompt / tokens_per_grid_unit)) then one decode record per output
// token (grid decode_grid), or `iterations` training records (grid
// train_grid; iterations <= 0 falls back to default_iterations).  Each record
// carries the lab seed mix_seed(job, position in job).
int ds_expand_workload(const ds_request* reqs, int64_t n_reqs, const ds_expand_params* p, ds_kernel_plan* out,
                       int64_t cap, int64_t* n) {
    if ((!reqs && n_reqs > 0) || !p || !n || cap < 0 || p->tokens_per_grid_unit <= 0) return DS_INVALID_ARGUMENT;
    std::map<int32_t, int32_t> job_of_stream;  // stream -> job (vctx) index
    std::map<int32_t, int32_t> kind_of_job;
    std::vector<int64_t> job_len;
    int64_t k = 0;
    auto push = [&](const ds_kernel_plan& e) {
        if (k < cap && out) out[k] = e;
        ++k;
    };
    for (int64_t r = 0; r < n_reqs; ++r) {
        const ds_request& q = reqs[r];
        auto it = job_of_stream.find(q.stream);
        if (it == job_of_stream.end()) {
            it = job_of_stream.emplace(q.stream, (int32_t)job_len.size()).first;
            kind_of_job[it->second] = q.kind;
            job_len.push_back(0);
        } else if (kind_of_job[it->second] != q.kind) {
            return DS_CONFIG_ERROR;  // "job mixes inference and training records"
        }
        const int32_t job = it->second;
        ds_kernel_plan e{};
        e.request = r;
        e.job = job;
        e.arrival_q = q.arrival_q;
        if (q.kind == DS_REQ_INFERENCE) {
            e.phase = DS_PREFILL;
            e.decode_index = -1;
            e.grid_size = (q.prompt_tokens + p->tokens_per_grid_unit - 1) / p->tokens_per_grid_unit;
            e.lab_seed = mix_seed((uint64_t)job, (uint64_t)job_len[job]++);
            push(e);
            for (int t = 0; t < q.output_tokens; ++t) {
                e.phase = DS_DECODE;
                e.decode_index = t;
                e.grid_size = p->decode_grid;
                e.lab_seed = mix_seed((uint64_t)job, (uint64_t)job_len[job]++);
                push(e);
            }
        } else {
            const int iters = q.iterations > 0 ? q.iterations : p->default_iterations;
            for (int i = 0; i < iters; ++i) {
                e.phase = DS_TRAINING;
                e.decode_index = -1;
                e.grid_size = p->train_grid;
                e.lab_seed = mix_seed((uint64_t)job, (uint64_t)job_len[job]++);
                push(e);
            }
        }
    }
    *n = k;
    return DS_OK;
}

}  // extern "C"
