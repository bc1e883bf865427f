// Library-internal helpers shared by the .cu translation units.
#pragma once
#include <cuda_runtime.h>
#include "meshlayers_b200.h"

int ml_fail(int code, const char* msg);
int ml_fail_cuda(cudaError_t e, const char* what);

#define ML_CUDA(call)                                            \
    do {                                                         \
        cudaError_t _e = (call);                                 \
        if (_e != cudaSuccess) return ml_fail_cuda(_e, #call);   \
    } while (0)

// Row-slab triangle list (raster.cu): list[0 .. *count) = indices of the triangles whose conservative raster row
// range meets [row0, row0 + rows), any order.  list: ntri ints, count: one zeroed u64 (both device).  For row-sharded
// atlases: every later per-triangle pass of a rank walks the list instead of all triangles.
int ml_slab_triangle_list(const void* tri_xy, int tri_dtype, long long ntri, long long row0, long long rows,
                          int* list, unsigned long long* count, cudaStream_t st);
// slabs of at most this fraction of the atlas height use the list
inline bool ml_slab_uses_list(long long rows, long long height, long long ntri) { return rows * 2 <= height && ntri >= 4096; }

#ifdef __CUDACC__
#include "common.cuh"
inline TeaParams ml_make_tea_params(const ml_tea_params* tp) {
    TeaParams p;
    p.ww = tp->ww; p.wh = tp->wh; p.eps = tp->eps;
    p.sfx = tp->sfx; p.sfy = tp->sfy; p.bx = tp->bx; p.by = tp->by;
    p.depth = tp->depth; p.shape = tp->shape;
    p.dw = tp->depth_w; p.dh = tp->depth_h; p.tw = tp->shape_w; p.th = tp->shape_h;
    p.eps_f32 = tp->eps_f32;
    return p;
}
#endif
