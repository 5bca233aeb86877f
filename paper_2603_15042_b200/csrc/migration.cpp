// Working-set migration across places: which regions a
// tenant must copy eagerly before it resumes on another place, which follow
// lazily, and the copy itself over NVLink (copy engines, peer to peer).
//   compute_migration_set  proj/src/runtime/migration.cpp:21-49
//   full_eager_set         proj/src/runtime/migration.cpp:51-58
// Regions are identified by id; a place is a bit of resident_mask (a pctx in
// the reference, a GPU for cross-device migration).  Orders follow the
// reference: eager sorted by region id (unique), lazy in ascending region id
// (the reference's std::map iteration order).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <map>
#include <vector>

#include "../../include/detshare/ds.h"

extern "C" {

int ds_compute_migration_set(const ds_region* ws, int n_ws, const int32_t* touched, int n_touched, int dst,
                             int32_t* eager, int* n_eager, uint64_t* eager_bytes, int32_t* lazy, int* n_lazy,
                             uint64_t* lazy_bytes) {
    if ((n_ws > 0 && !ws) || (n_touched > 0 && !touched) || !n_eager || !n_lazy || !eager_bytes || !lazy_bytes ||
        dst < 0 || dst >= 64)
        return DS_INVALID_ARGUMENT;
    std::map<int32_t, const ds_region*> set;
    for (int i = 0; i < n_ws; ++i) set[ws[i].id] = &ws[i];
    std::vector<int32_t> e;
    for (int i = 0; i < n_touched; ++i) {
        auto it = set.find(touched[i]);
        if (it == set.end()) return DS_TRACE_VIOLATION;  // touches a region outside the working set
        const ds_region& r = *it->second;
        if (r.dirty || !((r.resident_mask >> dst) & 1ull)) e.push_back(r.id);
    }
    std::sort(e.begin(), e.end());
    e.erase(std::unique(e.begin(), e.end()), e.end());
    uint64_t eb = 0;
    for (size_t i = 0; i < e.size(); ++i) {
        if (eager) eager[i] = e[i];
        eb += set[e[i]]->bytes;
    }
    int nl = 0;
    uint64_t lb = 0;
    for (const auto& [id, r] : set) {
        if (!r->dirty || std::binary_search(e.begin(), e.end(), id)) continue;
        if (lazy) lazy[nl] = id;
        ++nl;
        lb += r->bytes;
    }
    *n_eager = (int)e.size();
    *eager_bytes = eb;
    *n_lazy = nl;
    *lazy_bytes = lb;
    return DS_OK;
}

int ds_full_eager_set(const ds_region* ws, int n_ws, int32_t* eager, int* n_eager, uint64_t* eager_bytes) {
    if ((n_ws > 0 && !ws) || !n_eager || !eager_bytes) return DS_INVALID_ARGUMENT;
    std::map<int32_t, uint64_t> set;
    for (int i = 0; i < n_ws; ++i) set[ws[i].id] = ws[i].bytes;
    int k = 0;
    uint64_t b = 0;
    for (const auto& [id, bytes] : set) {
        if (eager) eager[k] = id;
        ++k;
        b += bytes;
    }
    *n_eager = k;
    *eager_bytes = b;
    return DS_OK;
}

// The eager copy: region i from src_ptrs[i] on src_device to dst_ptrs[i] on
// dst_device, peer to peer over NVLink by the copy engines (no SMs: the
// destination's resident executor keeps running), enqueued on `stream` of
// the destination device; completes when the stream does.
int ds_migrate_regions(int src_device, int dst_device, const void* const* src_ptrs, void* const* dst_ptrs,
                       const uint64_t* bytes, int n, void* stream) {
    if (n < 0 || (n > 0 && (!src_ptrs || !dst_ptrs || !bytes))) return DS_INVALID_ARGUMENT;
    if (cudaSetDevice(dst_device) != cudaSuccess) return DS_NO_DEVICE;
    if (src_device != dst_device) {
        int can = 0;
        if (cudaDeviceCanAccessPeer(&can, dst_device, src_device) != cudaSuccess) return DS_CUDA_ERROR;
        if (can) {
            cudaError_t e = cudaDeviceEnablePeerAccess(src_device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return DS_CUDA_ERROR;
            cudaGetLastError();
        }
    }
    for (int i = 0; i < n; ++i) {
        if (cudaMemcpyPeerAsync(dst_ptrs[i], dst_device, src_ptrs[i], src_device, bytes[i], (cudaStream_t)stream) !=
            cudaSuccess)
            return DS_CUDA_ERROR;
    }
    return DS_OK;
}

}  // extern "C"
