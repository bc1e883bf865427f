// Per-texel kernels that run over the cached triangle-id map:
//   ml_surface_resolve : position / normal / area map (north star (1); oracle ext_surface_map)
//   ml_tea_texels      : the paper's projective brush (TEA) evaluated per texel for the owner
//                        triangle -- bit-identical to the per-triangle reference loop
//                        (KN:135-203) when uv islands do not overlap (SURVEY.md 8 note N1).
// One thread per texel, consecutive threads on consecutive texels of a row: the 4-byte id read
// is a coalesced stream; the triangle records are gathers that hit L1/L2 because neighbouring
// texels share their owner.
#include "common.cuh"
#include "meshlayers_b200.h"
#include "internal.h"

namespace {

constexpr int BLOCK = 256;

template <typename T>
__global__ void __launch_bounds__(BLOCK)
resolve_kernel(const T* __restrict__ tri_xy, const T* __restrict__ tri_pos, const T* __restrict__ tri_nrm,
               long long width, long long row0, long long n, const int* __restrict__ tri_id,
               float* __restrict__ pos, float* __restrict__ nrm, float* __restrict__ area,
               unsigned long long* covered) {
    long long cnt = 0;
    const long long stride = (long long)gridDim.x * BLOCK;
    for (long long i = (long long)blockIdx.x * BLOCK + threadIdx.x; i < n; i += stride) {
        const int t = tri_id[i];
        if (t < 0) {
            const float qnan = __int_as_float(0x7fc00000);
            pos[i] = qnan; pos[n + i] = qnan; pos[2 * n + i] = qnan;
            nrm[i] = 0.f; nrm[n + i] = 0.f; nrm[2 * n + i] = 0.f;
            area[i] = 0.f;
            continue;
        }
        ++cnt;
        const long long yy = i / width;
        const int x = (int)(i - yy * width), y = (int)(row0 + yy);
        TriSetup s;
        tri_load_ccw(tri_xy + 6ll * t, s);
        double e0, e1, e2;
        tri_inside(s, x, y, e0, e1, e2);
        const double esum = xadd(xadd(e0, e1), e2);
        const double l0 = xdiv(e0, esum), l1 = xdiv(e1, esum), l2 = xdiv(e2, esum);
        const int i1 = s.swapped ? 6 : 3, i2 = s.swapped ? 3 : 6;
        const T* P = tri_pos + 9ll * t;
        const T* N = tri_nrm + 9ll * t;
        double p0[3], p1[3], p2[3], nv[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            p0[c] = (double)P[c]; p1[c] = (double)P[i1 + c]; p2[c] = (double)P[i2 + c];
            pos[c * n + i] = (float)xadd(xadd(xmul(l0, p0[c]), xmul(l1, p1[c])), xmul(l2, p2[c]));
            nv[c] = xadd(xadd(xmul(l0, (double)N[c]), xmul(l1, (double)N[i1 + c])), xmul(l2, (double)N[i2 + c]));
        }
        const double len = __dsqrt_rn(xadd(xadd(xmul(nv[0], nv[0]), xmul(nv[1], nv[1])), xmul(nv[2], nv[2])));
#pragma unroll
        for (int c = 0; c < 3; ++c) nrm[c * n + i] = (len > 0.0) ? (float)xdiv(nv[c], len) : 0.f;
        const double ux = xsub(p1[0], p0[0]), uy = xsub(p1[1], p0[1]), uz = xsub(p1[2], p0[2]);
        const double vx = xsub(p2[0], p0[0]), vy = xsub(p2[1], p0[1]), vz = xsub(p2[2], p0[2]);
        const double crx = xsub(xmul(uy, vz), xmul(uz, vy));
        const double cry = xsub(xmul(uz, vx), xmul(ux, vz));
        const double crz = xsub(xmul(ux, vy), xmul(uy, vx));
        const double a3 = xmul(__dsqrt_rn(xadd(xadd(xmul(crx, crx), xmul(cry, cry)), xmul(crz, crz))), 0.5);
        // |area2| of the CCW-normalised triangle: swapping two vertices negates KN:35 exactly
        const double area2 = xsub(xmul(s.cx, xsub(s.y2, s.y0)), xmul(s.cy, xsub(s.x2, s.x0)));
        const double a2 = xmul(fabs(area2), 0.5);
        area[i] = (float)xdiv(a3, a2);
    }
    block_count_add(cnt, covered);
}

template <typename T>
__global__ void __launch_bounds__(BLOCK)
tea_texel_kernel(const T* __restrict__ tri_xy, const T* __restrict__ tri_clip, long long width,
                 long long row0, long long n, const int* __restrict__ tri_id, TeaParams p,
                 void* __restrict__ data, int esize, uint32_t value,
                 uint8_t* __restrict__ mask, uint8_t* __restrict__ edited,
                 unsigned long long* counters) {
    long long newly = 0, frags = 0;
    const long long stride = (long long)gridDim.x * BLOCK;
    for (long long i = (long long)blockIdx.x * BLOCK + threadIdx.x; i < n; i += stride) {
        const int t = tri_id[i];
        if (t < 0) continue;
        ++frags;
        const long long yy = i / width;
        const int x = (int)(i - yy * width), y = (int)(row0 + yy);
        TriSetup s;
        tri_load_ccw(tri_xy + 6ll * t, s);
        double e0, e1, e2;
        tri_inside(s, x, y, e0, e1, e2);
        const T* c = tri_clip + 12ll * t;
        const int i1 = s.swapped ? 8 : 4, i2 = s.swapped ? 4 : 8;
        double c0[4], c1[4], c2[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) { c0[k] = (double)c[k]; c1[k] = (double)c[i1 + k]; c2[k] = (double)c[i2 + k]; }
        if (!tea_fragment(p, e0, e1, e2, c0, c1, c2)) continue;
        // exactly one thread owns texel i in this kernel: plain read-modify-write is race-free
        if (edited[i] == 0) ++newly;                                     // KN:198-199
        store_value(data, esize, i, value);                              // KN:200
        mask[i] = 1;                                                     // KN:201
        edited[i] = 1;                                                   // KN:202
    }
    block_count_add(newly, counters);
    block_count_add(frags, counters + 1);
}

inline unsigned grid_for(long long n) {
    long long blocks = (n + BLOCK - 1) / BLOCK;
    const long long cap = (long long)ml_sm_count() * 32;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (unsigned)blocks;
}

}  // namespace

extern "C" {

int ml_surface_resolve(const void* tri_xy, const void* tri_pos, const void* tri_nrm, int tri_dtype,
                       int64_t ntri, int64_t width, int64_t row0, int64_t rows,
                       const int32_t* tri_id, float* pos, float* nrm, float* area,
                       uint64_t* covered, void* stream) {
    (void)ntri;
    cudaStream_t st = (cudaStream_t)stream;
    const long long n = (long long)rows * width;
    if (n <= 0) return ML_OK;
    unsigned long long* ctr = (unsigned long long*)covered;
    if (tri_dtype == ML_F32)
        resolve_kernel<float><<<grid_for(n), BLOCK, 0, st>>>((const float*)tri_xy, (const float*)tri_pos,
            (const float*)tri_nrm, width, row0, n, tri_id, pos, nrm, area, ctr);
    else if (tri_dtype == ML_F64)
        resolve_kernel<double><<<grid_for(n), BLOCK, 0, st>>>((const double*)tri_xy, (const double*)tri_pos,
            (const double*)tri_nrm, width, row0, n, tri_id, pos, nrm, area, ctr);
    else
        return ml_fail(ML_ERR_ARG, "tri_dtype must be ML_F32 or ML_F64");
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int ml_tea_texels(const void* tri_xy, const void* tri_clip, int tri_dtype, int64_t ntri,
                  int64_t width, int64_t row0, int64_t rows, const int32_t* tri_id,
                  const ml_tea_params* tp, void* data, int esize, uint32_t value_bits,
                  uint8_t* mask, uint8_t* edited, uint64_t* counters, void* stream) {
    (void)ntri;
    cudaStream_t st = (cudaStream_t)stream;
    if (esize != 1 && esize != 2 && esize != 4) return ml_fail(ML_ERR_ARG, "esize must be 1, 2 or 4");
    const long long n = (long long)rows * width;
    if (n <= 0) return ML_OK;
    TeaParams p = ml_make_tea_params(tp);
    unsigned long long* ctr = (unsigned long long*)counters;
    if (tri_dtype == ML_F32)
        tea_texel_kernel<float><<<grid_for(n), BLOCK, 0, st>>>((const float*)tri_xy, (const float*)tri_clip,
            width, row0, n, tri_id, p, data, esize, value_bits, mask, edited, ctr);
    else if (tri_dtype == ML_F64)
        tea_texel_kernel<double><<<grid_for(n), BLOCK, 0, st>>>((const double*)tri_xy, (const double*)tri_clip,
            width, row0, n, tri_id, p, data, esize, value_bits, mask, edited, ctr);
    else
        return ml_fail(ML_ERR_ARG, "tri_dtype must be ML_F32 or ML_F64");
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

}  // extern "C"
