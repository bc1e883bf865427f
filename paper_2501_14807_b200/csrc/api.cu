// Library plumbing (errors, device query) and the host-buffer forms of the octree baseline kernels.
// The host-buffer twins of the hot path (KN:84, 103, 135-136) live in hostpath.cu.
#include <stdio.h>
#include <string.h>
#include <math.h>
#include "internal.h"

namespace {
thread_local char g_err[512] = "";
int g_sm_count = 0;
}

int ml_fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

int ml_fail_cuda(cudaError_t e, const char* what) {
    snprintf(g_err, sizeof g_err, "CUDA error %d (%s) at %s", (int)e, cudaGetErrorString(e), what);
    return e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ? ML_ERR_NO_DEVICE : ML_ERR_CUDA;
}

namespace {

// RAII device buffer for the host entry points
struct DevBuf {
    void* p = nullptr;
    ~DevBuf() { if (p) cudaFree(p); }
    cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 1); }
    template <typename T> T* as() { return (T*)p; }
};

#define ML_TRY(call) do { int _rc = (call); if (_rc != ML_OK) return _rc; } while (0)

}  // namespace

extern "C" {

int ml_version(void) { return 100; }

const char* ml_last_error(void) { return g_err; }

int ml_sm_count(void) {
    if (g_sm_count > 0) return g_sm_count;
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    g_sm_count = n;
    return n;
}

// KN:303-329 with host buffers.  *count = number of (cell, triangle) rows the expansion produces;
// they are written only when count <= capacity (the caller re-calls with a larger buffer otherwise).
int ml_expand_pairs_ordered_host(const double* verts, int64_t nverts, const int32_t* tris, int64_t ntri,
                                 const uint32_t* parent_cells, int64_t nparents, const int32_t* pair_parent,
                                 const int32_t* pair_tri, int64_t npair, const double* cube_min, double child_h,
                                 uint32_t* out_cells, int32_t* out_tri, int64_t capacity, int64_t* count) {
    if (!count) return ml_fail(ML_ERR_ARG, "ml_expand_pairs_ordered_host: count is required");
    *count = 0;
    if (npair <= 0) return ML_OK;                                    // KN:307-309
    if (nverts <= 0 || ntri <= 0 || nparents <= 0)
        return ml_fail(ML_ERR_ARG, "ml_expand_pairs_ordered_host: pairs without mesh / parent cells");
    if (ml_sm_count() <= 0) return ml_fail(ML_ERR_NO_DEVICE, "no CUDA device");
    const size_t ws = ml_expand_pairs_workspace_bytes(npair);
    DevBuf d_v, d_t, d_pc, d_pp, d_pt, d_ws, d_tot, d_oc, d_ot;
    ML_CUDA(d_v.alloc((size_t)nverts * 3 * sizeof(double)));
    ML_CUDA(d_t.alloc((size_t)ntri * 3 * sizeof(int32_t)));
    ML_CUDA(d_pc.alloc((size_t)nparents * 3 * sizeof(uint32_t)));
    ML_CUDA(d_pp.alloc((size_t)npair * sizeof(int32_t)));
    ML_CUDA(d_pt.alloc((size_t)npair * sizeof(int32_t)));
    ML_CUDA(d_ws.alloc(ws));
    ML_CUDA(d_tot.alloc(sizeof(uint64_t)));
    ML_CUDA(cudaMemcpyAsync(d_v.p, verts, (size_t)nverts * 3 * sizeof(double), cudaMemcpyHostToDevice, 0));
    ML_CUDA(cudaMemcpyAsync(d_t.p, tris, (size_t)ntri * 3 * sizeof(int32_t), cudaMemcpyHostToDevice, 0));
    ML_CUDA(cudaMemcpyAsync(d_pc.p, parent_cells, (size_t)nparents * 3 * sizeof(uint32_t), cudaMemcpyHostToDevice, 0));
    ML_CUDA(cudaMemcpyAsync(d_pp.p, pair_parent, (size_t)npair * sizeof(int32_t), cudaMemcpyHostToDevice, 0));
    ML_CUDA(cudaMemcpyAsync(d_pt.p, pair_tri, (size_t)npair * sizeof(int32_t), cudaMemcpyHostToDevice, 0));
    ML_TRY(ml_expand_pairs_count(d_v.as<double>(), d_t.as<int32_t>(), d_pc.as<uint32_t>(), d_pp.as<int32_t>(),
                                 d_pt.as<int32_t>(), npair, cube_min, child_h, d_ws.p, ws, d_tot.as<uint64_t>(),
                                 nullptr));
    uint64_t total = 0;
    ML_CUDA(cudaMemcpy(&total, d_tot.p, sizeof total, cudaMemcpyDeviceToHost));
    *count = (int64_t)total;
    if (total == 0 || (int64_t)total > capacity) return ML_OK;
    if (!out_cells || !out_tri) return ml_fail(ML_ERR_ARG, "ml_expand_pairs_ordered_host: null output");
    ML_CUDA(d_oc.alloc((size_t)total * 3 * sizeof(uint32_t)));
    ML_CUDA(d_ot.alloc((size_t)total * sizeof(int32_t)));
    ML_TRY(ml_expand_pairs_emit(d_pc.as<uint32_t>(), d_pp.as<int32_t>(), d_pt.as<int32_t>(), npair, d_ws.p,
                                d_oc.as<uint32_t>(), d_ot.as<int32_t>(), nullptr));
    ML_CUDA(cudaMemcpyAsync(out_cells, d_oc.p, (size_t)total * 3 * sizeof(uint32_t), cudaMemcpyDeviceToHost, 0));
    ML_CUDA(cudaMemcpyAsync(out_tri, d_ot.p, (size_t)total * sizeof(int32_t), cudaMemcpyDeviceToHost, 0));
    ML_CUDA(cudaStreamSynchronize(0));
    return ML_OK;
}

// KN:361-525 with host buffers
int ml_raycast_host(const double* origins, const double* dirs, int64_t nrays, const uint64_t* keys, int64_t nkeys,
                    const int64_t* offsets, const int32_t* tri_idx, const double* verts, int64_t nverts,
                    const int32_t* tris, int64_t ntri, const double* cube_min, double h, int64_t n_cells,
                    const uint8_t* coarse, int64_t coarse_side, int coarse_shift,
                    double* best_t, int32_t* best_tri, int64_t* leaf_pos) {
    if (nrays <= 0) return ML_OK;
    if (nkeys < 0 || nverts < 0 || ntri < 0) return ml_fail(ML_ERR_ARG, "ml_raycast_host: negative size");
    if (ml_sm_count() <= 0) return ml_fail(ML_ERR_NO_DEVICE, "no CUDA device");
    int64_t nidx = 0;
    if (nkeys > 0) nidx = offsets[nkeys];
    const size_t csz = coarse ? (size_t)coarse_side * coarse_side * coarse_side : 0;
    DevBuf d_o, d_d, d_k, d_off, d_idx, d_v, d_t, d_c, d_bt, d_btri, d_leaf;
    ML_CUDA(d_o.alloc((size_t)nrays * 3 * sizeof(double)));
    ML_CUDA(d_d.alloc((size_t)nrays * 3 * sizeof(double)));
    ML_CUDA(d_k.alloc((size_t)nkeys * sizeof(uint64_t)));
    ML_CUDA(d_off.alloc((size_t)(nkeys + 1) * sizeof(int64_t)));
    ML_CUDA(d_idx.alloc((size_t)nidx * sizeof(int32_t)));
    ML_CUDA(d_v.alloc((size_t)nverts * 3 * sizeof(double)));
    ML_CUDA(d_t.alloc((size_t)ntri * 3 * sizeof(int32_t)));
    ML_CUDA(d_c.alloc(csz));
    ML_CUDA(d_bt.alloc((size_t)nrays * sizeof(double)));
    ML_CUDA(d_btri.alloc((size_t)nrays * sizeof(int32_t)));
    ML_CUDA(d_leaf.alloc((size_t)nrays * sizeof(int64_t)));
    ML_CUDA(cudaMemcpyAsync(d_o.p, origins, (size_t)nrays * 3 * sizeof(double), cudaMemcpyHostToDevice, 0));
    ML_CUDA(cudaMemcpyAsync(d_d.p, dirs, (size_t)nrays * 3 * sizeof(double), cudaMemcpyHostToDevice, 0));
    if (nkeys > 0) {
        ML_CUDA(cudaMemcpyAsync(d_k.p, keys, (size_t)nkeys * sizeof(uint64_t), cudaMemcpyHostToDevice, 0));
        ML_CUDA(cudaMemcpyAsync(d_off.p, offsets, (size_t)(nkeys + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, 0));
        ML_CUDA(cudaMemcpyAsync(d_idx.p, tri_idx, (size_t)nidx * sizeof(int32_t), cudaMemcpyHostToDevice, 0));
        ML_CUDA(cudaMemcpyAsync(d_v.p, verts, (size_t)nverts * 3 * sizeof(double), cudaMemcpyHostToDevice, 0));
        ML_CUDA(cudaMemcpyAsync(d_t.p, tris, (size_t)ntri * 3 * sizeof(int32_t), cudaMemcpyHostToDevice, 0));
    }
    if (csz) ML_CUDA(cudaMemcpyAsync(d_c.p, coarse, csz, cudaMemcpyHostToDevice, 0));
    ML_TRY(ml_raycast(d_o.as<double>(), d_d.as<double>(), nrays, d_k.as<uint64_t>(), nkeys, d_off.as<int64_t>(),
                      d_idx.as<int32_t>(), d_v.as<double>(), d_t.as<int32_t>(), cube_min, h, n_cells,
                      coarse ? d_c.as<uint8_t>() : nullptr, coarse_side, coarse_shift, d_bt.as<double>(),
                      d_btri.as<int32_t>(), d_leaf.as<int64_t>(), nullptr));
    ML_CUDA(cudaMemcpyAsync(best_t, d_bt.p, (size_t)nrays * sizeof(double), cudaMemcpyDeviceToHost, 0));
    ML_CUDA(cudaMemcpyAsync(best_tri, d_btri.p, (size_t)nrays * sizeof(int32_t), cudaMemcpyDeviceToHost, 0));
    ML_CUDA(cudaMemcpyAsync(leaf_pos, d_leaf.p, (size_t)nrays * sizeof(int64_t), cudaMemcpyDeviceToHost, 0));
    ML_CUDA(cudaStreamSynchronize(0));
    return ML_OK;
}

}  // extern "C"
