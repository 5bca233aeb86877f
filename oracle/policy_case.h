/* ORACLE / TEST INFRASTRUCTURE — a flat, language-neutral policy snapshot.
 *
 * One `pc_case` describes a PolicyView (policy.hpp:24-69), a LaunchContext
 * (policy.hpp:71-78), the predictor's observations (predictor.cpp:14-25) and
 * the policy config (policies.hpp:12-18).  tests/cpp/policy_diff.cpp builds
 * the B200 runtime's view from it (csrc/policy.hpp) and the reference's view
 * (ref_policy_eval in oracle/ref_harness.cpp, reference policies.cpp) and
 * compares every hook's decision.
 *
 * Signatures are indices into a fixed table: sig i = (PC_SIG_NAMES[i / 2],
 * grid (i & 1) ? 128 : 256). */
#pragma once
#include <stdint.h>

#define PC_MAXP 12
#define PC_MAXV 10
#define PC_MAXO 8
#define PC_MAXQ 3
#define PC_NSIG 8

static const char* const PC_SIG_NAMES[4] = {"decode", "prefill", "train", "other"};

typedef struct pc_pctx {
    int32_t device, standby, bound /* -1: none */, available;
    int64_t tier_num, tier_den;
    int64_t running_kernel;  /* -1: none */
    int32_t running_sig, running_phase, running_priority, n_queued;
    int64_t running_remaining;
    int32_t queued_sig[PC_MAXQ];
    int32_t pad;
    int64_t queued_hint[PC_MAXQ];
} pc_pctx;

typedef struct pc_vctx {
    int32_t priority, quarantined, bound, head_phase, decoding, pad;
    int64_t pending;
} pc_vctx;

typedef struct pc_case {
    int32_t policy; /* 0 slo-aware, 1 tpot-first, 2 temporal, 3 static */
    int32_t n_p, n_v, n_obs;
    int64_t quantum, now, active_vctx_count, cold_default;
    pc_pctx p[PC_MAXP];
    pc_vctx v[PC_MAXV];
    int32_t obs_sig[PC_MAXO];
    int64_t obs_dur[PC_MAXO];
    /* launch */
    int32_t l_vctx, l_has_kernel, l_sig, l_phase, l_has_slo, l_pad;
    int64_t l_base, l_sat_num, l_sat_den, l_request_arrival, l_ttft, l_tpot;
    /* static partition */
    int32_t n_assign;
    int32_t assign_v[PC_MAXV], assign_p[PC_MAXV];
} pc_case;

typedef struct pc_result {
    /* kind: 0 direct, 1 remap, 2 defer, 3 preempt, 4 no-action; target -1 = none */
    int32_t launch_kind, launch_target;
    int32_t congestion_kind, congestion_target;
    int32_t completion_kind, completion_target;
    int32_t order_key, has_review;
    int64_t review;
    int64_t hol[PC_MAXP];  /* predict_hol_blocking per pctx */
} pc_result;
