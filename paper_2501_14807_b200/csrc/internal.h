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
