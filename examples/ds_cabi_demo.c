/* Plain-C caller of the detshare C ABI (no Python, no torch): the binding a
 * corosim-side maintainer links against.  Host-only entry points, so it runs
 * on a CPU box too; tests/test_abi_cpu.py compiles and runs it.
 *
 *   cc -Iinclude examples/ds_cabi_demo.c -Lpaper_2603_15042_b200 -ldetshare -o /tmp/ds_demo
 *
 * 1. gen_burst (reference trace.cpp:204-232) -> a bursty request stream
 * 2. expand_workload (workload.cpp:51-174) -> kernel records per request
 * 3. place_tenants -> a 16-tenant mix partitioned over 8 GPUs
 * 4. compute_metrics (metrics.cpp:35-85) over request outcomes
 * 5. the error path: an invalid tier pool is refused with a status code
 *    (InvalidTier on a GPU host, create_pool types.cpp:87-98; NoDevice on a
 *    CPU host, where the device probe comes first). */
#include <stdio.h>
#include <stdlib.h>

#include "detshare/ds.h"

int main(void) {
    ds_request_template t = {DS_REQ_INFERENCE, 8, 64, 4, 16, 0, 2};
    int64_t n = 0;
    if (ds_gen_burst(1.0, 50.0, 2.0, 20.0, 100.0, &t, 0, NULL, 0, &n) != DS_OK) return 1;
    ds_request* reqs = (ds_request*)malloc(sizeof(ds_request) * (size_t)n);
    if (ds_gen_burst(1.0, 50.0, 2.0, 20.0, 100.0, &t, 0, reqs, n, &n) != DS_OK) return 1;
    ds_expand_params p = {8, 164, 2048, 50, 0};
    int64_t k = 0;
    if (ds_expand_workload(reqs, n, &p, NULL, 0, &k) != DS_OK) return 1;
    ds_kernel_plan* plan = (ds_kernel_plan*)malloc(sizeof(ds_kernel_plan) * (size_t)k);
    if (ds_expand_workload(reqs, n, &p, plan, k, &k) != DS_OK) return 1;
    printf("requests %lld first_arrival_q %lld kernels %lld first_grid %lld\n", (long long)n,
           (long long)reqs[0].arrival_q, (long long)k, (long long)plan[0].grid_size);

    ds_tenant_demand mix[16];
    for (int i = 0; i < 16; ++i) {
        int decode = i < 8;
        ds_tenant_demand d = {decode ? DS_LATENCY_CRITICAL : DS_BEST_EFFORT, decode ? DS_DECODE : DS_TRAINING,
                              decode ? 0.1 * (1 + i % 4) : 0.05, decode ? 0.02 : 0.2 * (1 + i % 4), 10.0};
        mix[i] = d;
    }
    int32_t where[16];
    if (ds_place_tenants(mix, 16, 8, 150.0, where) != DS_OK) return 1;
    printf("placement");
    for (int i = 0; i < 16; ++i) printf(" %d", where[i]);
    printf("\n");

    /* three requests: TTFT 5/7/9 us, TPOTs 10/3, 2, 4 us, SLO tpot 3.5 us */
    ds_request_outcome o[3] = {
        {1, 1, 4, 1, 0, 5000, 15000, 8000, 3500, 0},
        {1, 1, 2, 1, 1000, 8000, 10000, 8000, 3500, 0},
        {1, 1, 3, 1, 2000, 11000, 19000, 8000, 3500, 0},
    };
    ds_metrics m;
    if (ds_compute_metrics(o, 3, 20000, 0, &m) != DS_OK) return 1;
    printf("metrics ttft_p99 %lld/%lld tpot_p50 %lld/%lld tpot_violations %lld\n", (long long)m.ttft.p99_num,
           (long long)m.ttft.p99_den, (long long)m.tpot.p50_num, (long long)m.tpot.p50_den,
           (long long)m.tpot_violations);

    ds_domain_config bad = {0};
    bad.n_tiers = 1;
    bad.tier_num[0] = 3;
    bad.tier_den[0] = 2; /* 3/2 is outside (0, 1] */
    ds_domain* dom = NULL;
    int rc = ds_domain_create(&bad, &dom);
    printf("bad pool -> %s\n", ds_status_name(rc));
    free(plan);
    free(reqs);
    return 0;
}
