// Workload-aware placement of tenants onto GPUs (config 5).
//
// Each B200 is an independent sharing domain, so a tenant mix is partitioned
// across devices once, at registration.  The reference places a vctx by
// pick_bind_target over the pctxs of every device in pool order
// (proj/src/policy/policies.cpp:74-94) — first fit on compute tiers only.  On
// B200 the two resources that decide co-location quality are different per
// tenant class: decode is HBM-bound, training GEMMs are tensor-bound, so the
// placement balances a 2-D load vector per device:
//
//   order  : latency-critical first, then by dominant demand (desc), then index
//   choose : the device minimising max(hbm_load + t.hbm, tensor_load + t.tensor)
//            with a penalty for a second latency-critical tenant on a device
//            (TPOT-First gives LC tenants SMs first; two of them contend), among
//            devices whose resident memory stays within the cap
//   ties   : lowest device index (deterministic: every rank computes the same map)
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

#include "../../include/detshare/ds.h"

extern "C" int ds_place_tenants(const ds_tenant_demand* t, int n, int n_devices, double mem_cap_gb,
                                int32_t* device_out) {
    if ((n > 0 && (!t || !device_out)) || n < 0 || n_devices < 1) return DS_INVALID_ARGUMENT;
    for (int i = 0; i < n; ++i)
        if (t[i].hbm_frac < 0 || t[i].tensor_frac < 0 || t[i].mem_gb < 0) return DS_INVALID_ARGUMENT;
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    auto dominant = [&](int i) { return std::max(t[i].hbm_frac, t[i].tensor_frac); };
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        const bool la = t[a].priority == DS_LATENCY_CRITICAL, lb = t[b].priority == DS_LATENCY_CRITICAL;
        if (la != lb) return la;
        const double da = dominant(a), db = dominant(b);
        if (da != db) return da > db;
        return a < b;
    });
    std::vector<double> hbm(n_devices, 0.0), tensor(n_devices, 0.0), mem(n_devices, 0.0);
    std::vector<int> lc(n_devices, 0);
    for (int i : order) {
        const bool is_lc = t[i].priority == DS_LATENCY_CRITICAL;
        int best = -1;
        double best_cost = 0;
        for (int d = 0; d < n_devices; ++d) {
            if (mem_cap_gb > 0 && mem[d] + t[i].mem_gb > mem_cap_gb) continue;
            double cost = std::max(hbm[d] + t[i].hbm_frac, tensor[d] + t[i].tensor_frac);
            if (is_lc) cost += 1.0 * lc[d];  // spread latency-critical tenants first
            if (best < 0 || cost < best_cost - 1e-12) {
                best = d;
                best_cost = cost;
            }
        }
        if (best < 0) return DS_CONFIG_ERROR;  // no device has room for this tenant
        device_out[i] = best;
        hbm[best] += t[i].hbm_frac;
        tensor[best] += t[i].tensor_frac;
        mem[best] += t[i].mem_gb;
        lc[best] += is_lc ? 1 : 0;
    }
    return DS_OK;
}
