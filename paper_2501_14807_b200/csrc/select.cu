// Selection brushes (north star (2)): sphere brush over the position map and attribute-threshold
// selection.  No reference code exists for them; the frozen definitions are
// oracle/kn_port.c ext_select_sphere / ext_select_sphere_batch / ext_select_threshold, and the
// write rule is the reference's (KN:198-202: count 0 -> 1 edits, data = value, mask = 1,
// edited = 1).
//
// Both are pure HBM streams: 12 B/texel (three float32 position planes) resp. attr + valid bytes,
// read once with 128-bit no-allocate loads, UNROLL independent loads per plane in flight per
// thread.  Hits are written per 4-texel quad with 32-bit read-modify-writes (common.cuh
// quad_write), so hit-dense strokes do not degenerate into partial-sector byte stores.
#include <cuda_fp16.h>
#include <limits.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include "common.cuh"
#include "bulk.cuh"
#include "meshlayers_b200.h"
#include "internal.h"

namespace {

constexpr int BLOCK = 256;
constexpr int UNROLL = 4;
#ifndef ML_THR_TU
#define ML_THR_TU 4
#endif
constexpr int TU = ML_THR_TU;  // quads in flight per thread of the threshold kernel

ML_DEV void hit_write(void* data, int esize, uint32_t value, uint8_t* mask, uint8_t* edited,
                      long long i, long long& cnt) {
    if (edited[i] == 0) ++cnt;
    store_value(data, esize, i, value);
    mask[i] = 1;
    edited[i] = 1;
}

ML_DEV bool sphere_hit(double px, double py, double pz, double cx, double cy, double cz, double r2) {
    const double dx = xsub(px, cx), dy = xsub(py, cy), dz = xsub(pz, cz);
    const double d2 = xadd(xadd(xmul(dx, dx), xmul(dy, dy)), xmul(dz, dz));
    return d2 <= r2;
}

ML_DEV unsigned sphere_hits4(const float4& x, const float4& y, const float4& z,
                             double cx, double cy, double cz, double r2) {
    unsigned h = 0;
    if (sphere_hit((double)x.x, (double)y.x, (double)z.x, cx, cy, cz, r2)) h |= 1u;
    if (sphere_hit((double)x.y, (double)y.y, (double)z.y, cx, cy, cz, r2)) h |= 2u;
    if (sphere_hit((double)x.z, (double)y.z, (double)z.z, cx, cy, cz, r2)) h |= 4u;
    if (sphere_hit((double)x.w, (double)y.w, (double)z.w, cx, cy, cz, r2)) h |= 8u;
    return h;
}

// ES > 0: aligned quad path (planes 16-byte aligned); ES == 0: scalar fallback for any layout.
template <int ES>
__global__ void __launch_bounds__(BLOCK)
sphere_kernel(const float* __restrict__ px, const float* __restrict__ py, const float* __restrict__ pz,
              long long n, double cx, double cy, double cz, double r2,
              void* __restrict__ data, int esize, uint32_t value,
              uint8_t* __restrict__ mask, uint8_t* __restrict__ edited, unsigned long long* counter) {
    long long cnt = 0;
    const long long tid = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * BLOCK;
    long long done = 0;
    if (ES > 0) {
        const long long nq = n >> 2;
        const float4* qx = (const float4*)px; const float4* qy = (const float4*)py; const float4* qz = (const float4*)pz;
        for (long long q0 = tid; q0 < nq; q0 += nthreads * UNROLL) {
            float4 vx[UNROLL], vy[UNROLL], vz[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const long long q = q0 + u * nthreads;
                if (q < nq) { vx[u] = ld_stream(qx + q); vy[u] = ld_stream(qy + q); vz[u] = ld_stream(qz + q); }
            }
            constexpr int E = ES > 0 ? ES : 1;
            unsigned hits[UNROLL];
            uint32_t ew[UNROLL], mw[UNROLL], dw[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u)
                hits[u] = (q0 + u * nthreads < nq) ? sphere_hits4(vx[u], vy[u], vz[u], cx, cy, cz, r2) : 0u;
#pragma unroll
            for (int u = 0; u < UNROLL; ++u)      // old words of all hit quads first: the loads overlap
                quad_load<E>(data, mask, edited, (q0 + u * nthreads) << 2, hits[u], ew[u], mw[u], dw[u]);
#pragma unroll
            for (int u = 0; u < UNROLL; ++u)
                quad_commit<E>(data, value, mask, edited, (q0 + u * nthreads) << 2, hits[u], ew[u], mw[u], dw[u], cnt);
        }
        done = nq << 2;
    }
    for (long long i = done + tid; i < n; i += nthreads)
        if (sphere_hit((double)px[i], (double)py[i], (double)pz[i], cx, cy, cz, r2))
            hit_write(data, esize, value, mask, edited, i, cnt);
    block_count_add(cnt, counter);
}

// ---------------------------------------------------------------------------------------------
// K strokes in one pass.  Work unit = one WARP x 512 consecutive texels (each lane holds 4 quads,
// every load instruction covers 512 contiguous bytes):
//   1. the warp streams its texels into registers and reduces their bounding box with shuffles;
//   2. strokes are culled 32 at a time (lane k tests stroke k0+k against the box, conservative
//      float64 sphere/box distance) into a ballot mask -- ascending bit order is stroke order;
//   3. every texel tests only the surviving strokes, in order, so the result equals K successive
//      single-stroke passes (a later stroke overwrites an earlier one on the same layer).
// No shared-memory lists and no block barriers in the loop; per-layer edit counts go to shared
// counters (L <= 64) and are flushed once per block.
struct BatchArgs {
    const float *px, *py, *pz;
    long long n;
    const double* strokes; const int* layer_of; const uint32_t* value_bits; long long K;
    void* const* data; uint8_t* const* mask; uint8_t* const* edited; long long L;
    unsigned long long* counts;
};

// conservative sphere / box test in float64: false only when NO point of the box [lo, hi] can pass
// d2 <= r*r.  Per-axis distance from the centre to the box: max(lo - c, c - hi, 0).  Every point p
// of the box has fl(d2(p)) >= dmin2*(1 - 8u): the box is provably missed only when
// dmin2 > r*r*(1 + 1e-12); otherwise the stroke is kept.
ML_DEV bool box_may_hit(double bl0, double bl1, double bl2, double bh0, double bh1, double bh2,
                        double sx, double sy, double sz, double sr) {
    const double ddx = fmax(fmax(xsub(bl0, sx), xsub(sx, bh0)), 0.0);
    const double ddy = fmax(fmax(xsub(bl1, sy), xsub(sy, bh1)), 0.0);
    const double ddz = fmax(fmax(xsub(bl2, sz), xsub(sz, bh2)), 0.0);
    const double dmin2 = xadd(xadd(xmul(ddx, ddx), xmul(ddy, ddy)), xmul(ddz, ddz));
    return !(dmin2 > xmul(xmul(sr, sr), 1.000000000001));
}

// All strokes of the batch against the 4 x 32 quads a warp holds in registers (quad u of lane l is
// texel 4*qidx[u]; qidx[u] < 0 = nothing).  Strokes are culled 32 at a time against the box of the
// held texels (lane k tests stroke k0+k) into a ballot mask -- ascending bit order is stroke order --
// and every texel tests only the survivors, in order, so the result equals K successive
// single-stroke passes (a later stroke overwrites an earlier one on the same layer).
template <int ES>
ML_DEV void batch_apply(const BatchArgs& a, const float4 (&vx)[4], const float4 (&vy)[4], const float4 (&vz)[4],
                        const long long (&qidx)[4], double bl0, double bl1, double bl2, double bh0, double bh1,
                        double bh2, int lane, bool smem_counts, unsigned long long* s_counts) {
    for (long long k0 = 0; k0 < a.K; k0 += 32) {
        const long long kk = k0 + lane;
        bool keep = false;
        if (kk < a.K)
            keep = box_may_hit(bl0, bl1, bl2, bh0, bh1, bh2, a.strokes[4 * kk], a.strokes[4 * kk + 1],
                               a.strokes[4 * kk + 2], a.strokes[4 * kk + 3]);
        unsigned live = __ballot_sync(0xffffffffu, keep);
        while (live) {
            const int b = __ffs(live) - 1;
            live &= live - 1;
            const long long k = k0 + b;
            const double sx = __ldg(a.strokes + 4 * k), sy = __ldg(a.strokes + 4 * k + 1),
                         sz = __ldg(a.strokes + 4 * k + 2), sr = __ldg(a.strokes + 4 * k + 3);
            const double r2 = xmul(sr, sr);
            unsigned hits[4];
            unsigned any = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                hits[u] = qidx[u] >= 0 ? sphere_hits4(vx[u], vy[u], vz[u], sx, sy, sz, r2) : 0u;
                any |= hits[u];
            }
            if (any) {
                const int layer = __ldg(a.layer_of + k);
                const uint32_t value = __ldg(a.value_bits + k);
                void* d = a.data[layer]; uint8_t* m = a.mask[layer]; uint8_t* ed = a.edited[layer];
                long long c = 0;
                uint32_t ew[4], mw[4], dw[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) quad_load<ES>(d, m, ed, qidx[u] << 2, hits[u], ew[u], mw[u], dw[u]);
#pragma unroll
                for (int u = 0; u < 4; ++u) quad_commit<ES>(d, value, m, ed, qidx[u] << 2, hits[u], ew[u], mw[u], dw[u], c);
                if (c) atomicAdd(smem_counts ? &s_counts[layer] : a.counts + layer, (unsigned long long)c);
            }
        }
    }
}

// box of the (NaN-free part of the) positions a warp holds, reduced over the warp
ML_DEV bool warp_box(const float4 (&vx)[4], const float4 (&vy)[4], const float4 (&vz)[4], float (&lo)[3], float (&hi)[3]) {
    const float inf = __int_as_float(0x7f800000);
    lo[0] = lo[1] = lo[2] = inf; hi[0] = hi[1] = hi[2] = -inf;
#pragma unroll
    for (int u = 0; u < 4; ++u) {                    // fminf / fmaxf drop NaNs (uncovered texels)
        lo[0] = fminf(lo[0], fminf(fminf(vx[u].x, vx[u].y), fminf(vx[u].z, vx[u].w)));
        hi[0] = fmaxf(hi[0], fmaxf(fmaxf(vx[u].x, vx[u].y), fmaxf(vx[u].z, vx[u].w)));
        lo[1] = fminf(lo[1], fminf(fminf(vy[u].x, vy[u].y), fminf(vy[u].z, vy[u].w)));
        hi[1] = fmaxf(hi[1], fmaxf(fmaxf(vy[u].x, vy[u].y), fmaxf(vy[u].z, vy[u].w)));
        lo[2] = fminf(lo[2], fminf(fminf(vz[u].x, vz[u].y), fminf(vz[u].z, vz[u].w)));
        hi[2] = fmaxf(hi[2], fmaxf(fmaxf(vz[u].x, vz[u].y), fmaxf(vz[u].z, vz[u].w)));
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo[c] = fminf(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
            hi[c] = fmaxf(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
        }
    }
    return lo[0] <= hi[0];                           // false: no covered texel (warp-uniform)
}

template <int ES>
__global__ void __launch_bounds__(BLOCK, 2)
sphere_batch_kernel(BatchArgs a) {
    __shared__ unsigned long long s_counts[64];
    const bool smem_counts = a.L <= 64;
    if (threadIdx.x < 64) s_counts[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long nq = a.n >> 2;                        // host guarantees n % 4 == 0
    const long long nunits = (nq + 127) >> 7;             // 128 quads = 512 texels per warp unit
    const long long nwarps = (long long)gridDim.x * (BLOCK / 32);
    for (long long unit = (long long)blockIdx.x * (BLOCK / 32) + (threadIdx.x >> 5); unit < nunits; unit += nwarps) {
        float4 vx[4], vy[4], vz[4];
        long long qidx[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long long q = (unit << 7) + u * 32 + lane;
            qidx[u] = q < nq ? q : -1;
            if (q < nq) {
                vx[u] = ld_stream((const float4*)a.px + q);
                vy[u] = ld_stream((const float4*)a.py + q);
                vz[u] = ld_stream((const float4*)a.pz + q);
            } else {
                const float qn = __int_as_float(0x7fc00000);
                vx[u] = vy[u] = vz[u] = make_float4(qn, qn, qn, qn);
            }
        }
        float lo[3], hi[3];
        if (!warp_box(vx, vy, vz, lo, hi)) continue;
        batch_apply<ES>(a, vx, vy, vz, qidx, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2], lane, smem_counts, s_counts);
    }
    __syncthreads();
    if (smem_counts && threadIdx.x < a.L && s_counts[threadIdx.x]) atomicAdd(a.counts + threadIdx.x, s_counts[threadIdx.x]);
}

// ---------------------------------------------------------------------------------------------
// Footprint-culled brushes.  The surface map carries one float32 bounding box per 128 x 4-texel
// TILE of the position planes (built once, ml_surface_tile_boxes: 32 bytes per 512 texels).  A
// stroke first tests the boxes (one thread per tile, conservative float64 test above) and appends
// the tiles it may touch to a list; a second launch walks the list with one warp per tile and runs
// exactly the per-texel test and write rule of the streaming kernels.  A stroke then costs
// O(tiles) * 32 B + O(footprint) * 12 B instead of 12 B for every texel of the atlas; the planes
// and counts are identical because a culled tile provably contains no hit.
constexpr int ST_W_SHIFT = 7, ST_H_SHIFT = 2;              // 128 texels x 4 rows

struct TileGrid {
    long long width, rows, nq;
    int segs, tile_rows;
    long long ntiles;
};
inline TileGrid tile_grid(long long width, long long rows) {
    TileGrid g;
    g.width = width; g.rows = rows; g.nq = (width * rows) >> 2;
    g.segs = (int)(width >> ST_W_SHIFT);
    g.tile_rows = (int)((rows + (1 << ST_H_SHIFT) - 1) >> ST_H_SHIFT);
    g.ntiles = (long long)g.segs * g.tile_rows;
    return g;
}
// quad index of (row u of the tile, lane) or -1 below the slab
ML_DEV long long tile_quad(const TileGrid& g, long long tile, int u, int lane) {
    const long long ty = tile / g.segs, tx = tile - ty * g.segs;
    const long long yy = (ty << ST_H_SHIFT) + u;
    return yy < g.rows ? ((yy * g.width + (tx << ST_W_SHIFT)) >> 2) + lane : -1;
}
ML_DEV void tile_load(const TileGrid& g, long long tile, int lane, const float* px, const float* py, const float* pz,
                      float4 (&vx)[4], float4 (&vy)[4], float4 (&vz)[4], long long (&qidx)[4]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        qidx[u] = tile_quad(g, tile, u, lane);
        if (qidx[u] >= 0) {
            vx[u] = ld_stream((const float4*)px + qidx[u]);
            vy[u] = ld_stream((const float4*)py + qidx[u]);
            vz[u] = ld_stream((const float4*)pz + qidx[u]);
        } else {
            const float qn = __int_as_float(0x7fc00000);
            vx[u] = vy[u] = vz[u] = make_float4(qn, qn, qn, qn);
        }
    }
}

__global__ void __launch_bounds__(BLOCK)
tile_box_kernel(const float* __restrict__ px, const float* __restrict__ py, const float* __restrict__ pz,
                TileGrid g, float4* __restrict__ boxes) {
    const int lane = threadIdx.x & 31;
    const long long nwarps = (long long)gridDim.x * (BLOCK / 32);
    for (long long tile = (long long)blockIdx.x * (BLOCK / 32) + (threadIdx.x >> 5); tile < g.ntiles; tile += nwarps) {
        float4 vx[4], vy[4], vz[4];
        long long qidx[4];
        tile_load(g, tile, lane, px, py, pz, vx, vy, vz, qidx);
        float lo[3], hi[3];
        warp_box(vx, vy, vz, lo, hi);                      // empty tile: lo = +inf > hi = -inf
        if (lane == 0) {
            boxes[2 * tile] = make_float4(lo[0], lo[1], lo[2], 0.f);
            boxes[2 * tile + 1] = make_float4(hi[0], hi[1], hi[2], 0.f);
        }
    }
}

// tile list in device scratch: [count u64][pad u64][bitmap ntiles/32 u32, rounded to 8 B][u32 tile indices]
struct TileList { unsigned long long* count; uint32_t* bits; uint32_t* tiles; };
inline long long tile_bitmap_words(long long ntiles) { return ((ntiles + 63) / 64) * 2; }

// One thread per (tile, chunk of KC strokes): blockIdx.y selects the chunk, so a batch of many
// strokes still fills the machine.  A tile is appended to the list by the first chunk that finds a
// stroke reaching it (atomicOr on the tile bitmap decides who appends).  K == 1 / strokes == NULL is
// the single-stroke brush.
constexpr int KC = 32;
__global__ void __launch_bounds__(BLOCK)
tile_classify_kernel(const float4* __restrict__ boxes, long long ntiles, const double* __restrict__ strokes,
                     long long K, double cx, double cy, double cz, double cr, TileList list) {
    const long long tile = (long long)blockIdx.x * BLOCK + threadIdx.x;
    if (tile >= ntiles) return;
    const uint32_t bit = 1u << (tile & 31);
    if (gridDim.y > 1 && (ld_volatile_u32(list.bits + (tile >> 5)) & bit)) return;      // another chunk already kept it
    const float4 lo = __ldg(boxes + 2 * tile), hi = __ldg(boxes + 2 * tile + 1);
    if (!(lo.x <= hi.x)) return;                                                        // no covered texel
    bool keep = false;
    if (strokes == nullptr) keep = box_may_hit(lo.x, lo.y, lo.z, hi.x, hi.y, hi.z, cx, cy, cz, cr);
    else {
        for (long long k0 = (long long)blockIdx.y * KC; k0 < K && !keep; k0 += (long long)gridDim.y * KC) {
            const long long k1 = k0 + KC < K ? k0 + KC : K;
            for (long long k = k0; k < k1 && !keep; ++k)
                keep = box_may_hit(lo.x, lo.y, lo.z, hi.x, hi.y, hi.z, __ldg(strokes + 4 * k), __ldg(strokes + 4 * k + 1),
                                   __ldg(strokes + 4 * k + 2), __ldg(strokes + 4 * k + 3));
        }
    }
    if (keep && !(atomicOr(list.bits + (tile >> 5), bit) & bit))
        list.tiles[atomicAdd(list.count, 1ull)] = (uint32_t)tile;
}

template <int ES>
__global__ void __launch_bounds__(BLOCK)
sphere_tiles_kernel(const float* __restrict__ px, const float* __restrict__ py, const float* __restrict__ pz,
                    TileGrid g, TileList list, double cx, double cy, double cz, double r2,
                    void* __restrict__ data, uint32_t value, uint8_t* __restrict__ mask,
                    uint8_t* __restrict__ edited, unsigned long long* counter) {
    long long cnt = 0;
    const int lane = threadIdx.x & 31;
    const long long count = (long long)*list.count;
    const long long nwarps = (long long)gridDim.x * (BLOCK / 32);
    for (long long j = (long long)blockIdx.x * (BLOCK / 32) + (threadIdx.x >> 5); j < count; j += nwarps) {
        float4 vx[4], vy[4], vz[4];
        long long qidx[4];
        tile_load(g, list.tiles[j], lane, px, py, pz, vx, vy, vz, qidx);
        unsigned hits[4];
        uint32_t ew[4], mw[4], dw[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) hits[u] = qidx[u] >= 0 ? sphere_hits4(vx[u], vy[u], vz[u], cx, cy, cz, r2) : 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u) quad_load<ES>(data, mask, edited, qidx[u] << 2, hits[u], ew[u], mw[u], dw[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) quad_commit<ES>(data, value, mask, edited, qidx[u] << 2, hits[u], ew[u], mw[u], dw[u], cnt);
    }
    block_count_add(cnt, counter);
}

template <int ES>
__global__ void __launch_bounds__(BLOCK, 2)
sphere_batch_tiles_kernel(BatchArgs a, TileGrid g, const float4* __restrict__ boxes, TileList list) {
    __shared__ unsigned long long s_counts[64];
    const bool smem_counts = a.L <= 64;
    if (threadIdx.x < 64) s_counts[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long count = (long long)*list.count;
    const long long nwarps = (long long)gridDim.x * (BLOCK / 32);
    for (long long j = (long long)blockIdx.x * (BLOCK / 32) + (threadIdx.x >> 5); j < count; j += nwarps) {
        const long long tile = list.tiles[j];
        float4 vx[4], vy[4], vz[4];
        long long qidx[4];
        tile_load(g, tile, lane, a.px, a.py, a.pz, vx, vy, vz, qidx);
        const float4 lo = __ldg(boxes + 2 * tile), hi = __ldg(boxes + 2 * tile + 1);
        batch_apply<ES>(a, vx, vy, vz, qidx, lo.x, lo.y, lo.z, hi.x, hi.y, hi.z, lane, smem_counts, s_counts);
    }
    __syncthreads();
    if (smem_counts && threadIdx.x < a.L && s_counts[threadIdx.x]) atomicAdd(a.counts + threadIdx.x, s_counts[threadIdx.x]);
}

// ---------------------------------------------------------------------------------------------
// The definition compares the attribute WIDENED TO FLOAT64 with [lo, hi].  Widening is exact for
// every plane kind, so the same decision can be taken in the attribute's own domain against
// thresholds rounded inward once on the host:  lo <= (double)a  <=>  a >= (smallest value of the
// kind that is >= lo), and likewise for hi.  NaN attributes fail both forms.  This removes all
// float64 conversions and compares from the stream.
struct Thr { float lo_f, hi_f; long long lo_i, hi_i; };

template <int KIND> struct AttrT;
template <> struct AttrT<ML_U8>  { typedef uint8_t T;  static ML_DEV bool hit(T v, const Thr& t) { return (long long)v >= t.lo_i && (long long)v <= t.hi_i; } static ML_DEV double get(T v) { return (double)v; } };
template <> struct AttrT<ML_I8>  { typedef int8_t T;   static ML_DEV bool hit(T v, const Thr& t) { return (long long)v >= t.lo_i && (long long)v <= t.hi_i; } static ML_DEV double get(T v) { return (double)v; } };
template <> struct AttrT<ML_I16> { typedef int16_t T;  static ML_DEV bool hit(T v, const Thr& t) { return (long long)v >= t.lo_i && (long long)v <= t.hi_i; } static ML_DEV double get(T v) { return (double)v; } };
template <> struct AttrT<ML_I32> { typedef int32_t T;  static ML_DEV bool hit(T v, const Thr& t) { return (long long)v >= t.lo_i && (long long)v <= t.hi_i; } static ML_DEV double get(T v) { return (double)v; } };
template <> struct AttrT<ML_U32> { typedef uint32_t T; static ML_DEV bool hit(T v, const Thr& t) { return (long long)v >= t.lo_i && (long long)v <= t.hi_i; } static ML_DEV double get(T v) { return (double)v; } };
template <> struct AttrT<ML_F16> { typedef uint16_t T; static ML_DEV bool hit(T v, const Thr& t) { const float f = __half2float(__ushort_as_half(v)); return f >= t.lo_f && f <= t.hi_f; } static ML_DEV double get(T v) { return (double)__half2float(__ushort_as_half(v)); } };
template <> struct AttrT<ML_FLOAT32> { typedef float T; static ML_DEV bool hit(T v, const Thr& t) { return v >= t.lo_f && v <= t.hi_f; } static ML_DEV double get(T v) { return (double)v; } };

// 4 texels per step: one (4*sizeof(T))-byte attribute load + one 4-byte valid load.
#ifndef ML_THR_MINB
#define ML_THR_MINB 4
#endif
template <int KIND, int ES>
__global__ void __launch_bounds__(BLOCK, ML_THR_MINB)
threshold_kernel(const void* __restrict__ attr_, const uint8_t* __restrict__ valid, long long n,
                 double lo, double hi, Thr thr, void* __restrict__ data, int esize, uint32_t value,
                 uint8_t* __restrict__ mask, uint8_t* __restrict__ edited, unsigned long long* counter) {
    typedef typename AttrT<KIND>::T T;
    const T* attr = (const T*)attr_;
    long long cnt = 0;
    const long long tid = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * BLOCK;
    long long done = 0;
    if (ES > 0) {
        struct __align__(sizeof(T) * 4) Quad { T v[4]; };
        const long long nq = n >> 2;
        for (long long q0 = tid; q0 < nq; q0 += nthreads * TU) {
            Quad a[TU]; uint32_t vm[TU];
#pragma unroll
            for (int u = 0; u < TU; ++u) {
                const long long q = q0 + u * nthreads;
                if (q < nq) {
                    a[u] = ld_quad((const Quad*)attr + q);
                    vm[u] = valid ? ld_stream((const uint32_t*)valid + q) : 0x01010101u;
                }
            }
            constexpr int E = ES > 0 ? ES : 1;
            unsigned hits[TU];
            uint32_t ew[TU], mw[TU], dw[TU];
#pragma unroll
            for (int u = 0; u < TU; ++u) {
                hits[u] = 0;
                const long long q = q0 + u * nthreads;
                if (q >= nq) continue;
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if ((((vm[u] >> (8 * e)) & 0xffu) != 0) && AttrT<KIND>::hit(a[u].v[e], thr)) hits[u] |= 1u << e;
            }
#pragma unroll
            for (int u = 0; u < TU; ++u)      // old words of all hit quads first: the loads overlap
                quad_load<E>(data, mask, edited, (q0 + u * nthreads) << 2, hits[u], ew[u], mw[u], dw[u]);
#pragma unroll
            for (int u = 0; u < TU; ++u)
                quad_commit<E>(data, value, mask, edited, (q0 + u * nthreads) << 2, hits[u], ew[u], mw[u], dw[u], cnt);
        }
        done = nq << 2;
    }
    for (long long i = done + tid; i < n; i += nthreads) {
        if (valid && valid[i] == 0) continue;
        const double v = AttrT<KIND>::get(attr[i]);
        if (lo <= v && v <= hi) hit_write(data, esize, value, mask, edited, i, cnt);
    }
    block_count_add(cnt, counter);
}

// ---------------------------------------------------------------------------------------------
// Footprint-culled threshold selection for float32 attribute planes that do not change between
// selections (geometry-derived attributes such as height = pos.z): the plane carries its [min, max]
// per 128 x 4-texel tile (ml_plane_tile_range, NaN = "no value" dropped).  The tile test is exact in
// the attribute's own domain -- a texel hits iff lo_f <= v <= hi_f with the inward-rounded float
// thresholds of launch_threshold, so a tile with max < lo_f or min > hi_f holds no hit -- and kept
// tiles run the per-texel test and write rule of threshold_kernel.
__global__ void __launch_bounds__(BLOCK)
tile_range_kernel(const float* __restrict__ attr, TileGrid g, float2* __restrict__ ranges) {
    const int lane = threadIdx.x & 31;
    const float inf = __int_as_float(0x7f800000);
    const long long nwarps = (long long)gridDim.x * (BLOCK / 32);
    for (long long tile = (long long)blockIdx.x * (BLOCK / 32) + (threadIdx.x >> 5); tile < g.ntiles; tile += nwarps) {
        float lo = inf, hi = -inf;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long long q = tile_quad(g, tile, u, lane);
            if (q < 0) continue;
            const float4 v = ld_stream((const float4*)attr + q);
            lo = fminf(lo, fminf(fminf(v.x, v.y), fminf(v.z, v.w)));      // fminf / fmaxf drop NaNs
            hi = fmaxf(hi, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) ranges[tile] = make_float2(lo, hi);
    }
}

__global__ void __launch_bounds__(BLOCK)
range_classify_kernel(const float2* __restrict__ ranges, long long ntiles, float lo_f, float hi_f, TileList list) {
    const long long tile = (long long)blockIdx.x * BLOCK + threadIdx.x;
    bool keep = false;
    if (tile < ntiles) {
        const float2 r = __ldg(ranges + tile);
        keep = (r.x <= r.y) && !(r.y < lo_f) && !(r.x > hi_f);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (bal == 0) return;
    const int lane = threadIdx.x & 31;
    unsigned long long slot = 0;
    if (lane == 0) slot = atomicAdd(list.count, (unsigned long long)__popc(bal));
    slot = __shfl_sync(0xffffffffu, slot, 0);
    if (keep) list.tiles[slot + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)tile;
}

template <int ES>
__global__ void __launch_bounds__(BLOCK, 4)
threshold_tiles_kernel(const float* __restrict__ attr, const uint8_t* __restrict__ valid, TileGrid g, TileList list,
                       Thr thr, void* __restrict__ data, uint32_t value, uint8_t* __restrict__ mask,
                       uint8_t* __restrict__ edited, unsigned long long* counter) {
    long long cnt = 0;
    const int lane = threadIdx.x & 31;
    const long long count = (long long)*list.count;
    const long long nwarps = (long long)gridDim.x * (BLOCK / 32);
    for (long long j = (long long)blockIdx.x * (BLOCK / 32) + (threadIdx.x >> 5); j < count; j += nwarps) {
        const long long tile = list.tiles[j];
        long long q[4];
        float4 a[4];
        uint32_t vm[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            q[u] = tile_quad(g, tile, u, lane);
            if (q[u] >= 0) {
                a[u] = ld_stream((const float4*)attr + q[u]);
                vm[u] = valid ? ld_stream((const uint32_t*)valid + q[u]) : 0x01010101u;
            }
        }
        unsigned hits[4];
        uint32_t ew[4], mw[4], dw[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            hits[u] = 0;
            if (q[u] < 0) continue;
            const float v[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if ((((vm[u] >> (8 * e)) & 0xffu) != 0) && AttrT<ML_FLOAT32>::hit(v[e], thr)) hits[u] |= 1u << e;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) quad_load<ES>(data, mask, edited, q[u] << 2, hits[u], ew[u], mw[u], dw[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) quad_commit<ES>(data, value, mask, edited, q[u] << 2, hits[u], ew[u], mw[u], dw[u], cnt);
    }
    block_count_add(cnt, counter);
}

// 16-texel form of the tile walk (default; the quad form above serves a valid plane that is only 4-byte aligned).
// The attribute loads stay as they are -- row u of the tile, lane l = quad l: one coalesced 512-byte access per row --
// but the byte planes are written by OWNER lanes: lane L owns the 16 texels [16 (L & 7), +16) of row L >> 3, so
// edited / mask / data move as one 128-bit access per plane and lane (vec16_load / vec16_commit) instead of four
// 32-bit ones.  The 4 x 4 hit bits of a lane travel to the owners with 4 shuffles.
#ifndef ML_TTV_U
#define ML_TTV_U 1          // tiles per warp step; measured at 16k^2 (C3 window): U = 1 at 4 blocks/SM 0.112 ms, U = 2 at 3 / 4 / 2 blocks 0.122 / 0.128 / 0.131
#endif
#ifndef ML_TTV_MINB
#define ML_TTV_MINB 4
#endif
template <int ES, bool HV>
__global__ void __launch_bounds__(BLOCK, ML_TTV_MINB)
threshold_tiles_vec_kernel(const float* __restrict__ attr, const uint8_t* __restrict__ valid, TileGrid g, TileList list,
                           Thr thr, void* __restrict__ data, uint32_t value, uint8_t* __restrict__ mask,
                           uint8_t* __restrict__ edited, unsigned long long* counter) {
    constexpr int U = ML_TTV_U;
    long long cnt = 0;
    const int lane = threadIdx.x & 31;
    const int orow = lane >> 3, oseg = lane & 7;
    const long long count = (long long)*list.count;
    const long long nwarps = (long long)gridDim.x * (BLOCK / 32);
    long long j = (long long)blockIdx.x * (BLOCK / 32) + (threadIdx.x >> 5);
    long long tile[U];
#pragma unroll
    for (int t = 0; t < U; ++t) tile[t] = j + t * nwarps < count ? (long long)list.tiles[j + t * nwarps] : -1;
    for (; j < count; j += U * nwarps) {
        long long row_base[U], col[U];
        float4 a[U][4];
        uint4 vv[U];
#pragma unroll
        for (int t = 0; t < U; ++t) {
            const long long ty = tile[t] / g.segs, tx = tile[t] - ty * g.segs;
            row_base[t] = tile[t] >= 0 ? ty << ST_H_SHIFT : g.rows;          // no tile: every row is "below the slab"
            col[t] = tx << ST_W_SHIFT;
            const long long jn = j + (U + t) * nwarps;
            tile[t] = jn < count ? (long long)list.tiles[jn] : -1;           // next step's tile: off the dependent-load chain
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (row_base[t] + u < g.rows)
                    a[t][u] = ld_stream((const float4*)attr + ((((row_base[t] + u) * g.width + col[t]) >> 2) + lane));
            vv[t] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
            if (HV && row_base[t] + orow < g.rows)
                vv[t] = ld_stream((const uint4*)(valid + (row_base[t] + orow) * g.width + col[t] + 16 * oseg));
        }
        unsigned hit16[U];
        uint4 ew[U], mw[U], dw[U];
#pragma unroll
        for (int t = 0; t < U; ++t) {
            unsigned packed = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (row_base[t] + u >= g.rows) continue;
                const float v[4] = {a[t][u].x, a[t][u].y, a[t][u].z, a[t][u].w};
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (AttrT<ML_FLOAT32>::hit(v[e], thr)) packed |= 1u << (4 * u + e);
            }
            hit16[t] = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const unsigned v = __shfl_sync(0xffffffffu, packed, 4 * oseg + k);
                hit16[t] |= ((v >> (4 * orow)) & 0xfu) << (4 * k);
            }
            if (HV) hit16[t] &= nz_bits4(vv[t].x) | (nz_bits4(vv[t].y) << 4) | (nz_bits4(vv[t].z) << 8) | (nz_bits4(vv[t].w) << 12);
            if (row_base[t] + orow >= g.rows) hit16[t] = 0;
            vec16_load<ES>(data, mask, edited, (row_base[t] + orow) * g.width + col[t] + 16 * oseg, hit16[t], ew[t], mw[t], dw[t]);
        }
#pragma unroll
        for (int t = 0; t < U; ++t)
            vec16_commit<ES>(data, value, mask, edited, (row_base[t] + orow) * g.width + col[t] + 16 * oseg, hit16[t],
                             ew[t], mw[t], dw[t], cnt);
    }
    block_count_add(cnt, counter);
}

// 16-texel form (default when attribute, valid and layer planes are 16-byte aligned).  A warp owns
// 512 consecutive texels per step.  The ATTRIBUTE bytes are fetched lane-interleaved -- load k of
// lane l is the 16-byte chunk k*32 + l of the warp's 512*S attribute bytes, so every load
// instruction is one fully coalesced 512-byte access -- and the chunk hit bits are then moved with S
// shuffles to the lane that owns the texels in BYTE-plane order (lane L owns texels 16L .. 16L+15),
// where valid / edited / mask / data move as one 128-bit access per plane (vec16_load / _commit).
// Compared with the quad form: the same attribute loads, a quarter of the byte-plane memory
// instructions, and VT * S * 16 bytes in flight per thread.
#ifndef ML_THR_VEC_MINB
#define ML_THR_VEC_MINB 3
#endif
#ifndef ML_THR_PIPE
#define ML_THR_PIPE 0
#endif
#ifndef ML_THR_WAVES
#define ML_THR_WAVES 1      // grid = resident blocks x this
#endif
template <int KIND, int ES, bool HV = true>
struct ThrTile {                               // one warp tile (512 texels) as held by one lane; HV: a valid plane exists
    typedef typename AttrT<KIND>::T T;
    static constexpr int S = (int)sizeof(T);   // 16-byte attribute chunks per 16 texels
    static constexpr int EPC = 16 / S;         // texels per chunk
    struct __align__(16) Chunk { T v[EPC]; };
    Chunk a[S];
    uint4 vm;

    // issue the tile's loads: S lane-interleaved attribute chunks (+ the valid bytes of this lane's vector)
    ML_DEV void load(const T* attr, const uint8_t* valid, long long tile, long long nv, int lane) {
        const long long vec = (tile << 5) + lane;
        vm = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
        if (valid && vec < nv) vm = ld_stream((const uint4*)valid + vec);
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const long long chunk = (tile << 5) * S + k * 32 + lane;
            uint4 w = make_uint4(0u, 0u, 0u, 0u);
            if (chunk < nv * S) w = ld_stream((const uint4*)attr + chunk);
            memcpy(&a[k], &w, 16);
        }
    }
    // same from a shared-memory copy of the tile's attribute bytes (`tile_smem`), of which `avail` bytes exist
    ML_DEV void load_smem(const uint8_t* tile_smem, unsigned avail, const uint8_t* valid, long long tile, long long nv, int lane) {
        const long long vec = (tile << 5) + lane;
        vm = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
        if (HV && valid && vec < nv) vm = ld_stream((const uint4*)valid + vec);
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const unsigned off = (unsigned)(k * 32 + lane) << 4;
            uint4 w = make_uint4(0u, 0u, 0u, 0u);
            if (off < avail) w = *(const uint4*)(tile_smem + off);
            memcpy(&a[k], &w, 16);
        }
    }
    // hit bits of this lane's 16 texels (byte-plane order) from the lane-interleaved chunks
    ML_DEV unsigned hits(const Thr& thr, long long tile, long long nv, int lane) const {
        unsigned pk = 0;                       // S fields of EPC hit bits, field k = chunk k*32 + lane
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const long long chunk = (tile << 5) * S + k * 32 + lane;
            unsigned h = 0;
            if (chunk < nv * S) {
#pragma unroll
                for (int e = 0; e < EPC; ++e) if (AttrT<KIND>::hit(a[k].v[e], thr)) h |= 1u << e;
            }
            pk |= h << (k * EPC);
        }
        // lane L's texels 16L .. 16L+15 are chunks L*S + j (j < S): load (L*S + j) / 32 of lane (L*S + j) % 32
        unsigned mine = 0;
        if (S == 1) mine = pk;
        else {
#pragma unroll
            for (int j = 0; j < S; ++j) {
                const int ci = lane * S + j;
                const unsigned got = __shfl_sync(0xffffffffu, pk, ci & 31);
                mine |= ((got >> ((ci >> 5) * EPC)) & ((1u << EPC) - 1u)) << (j * EPC);
            }
        }
        unsigned vbits = 0xffffu;
        if (HV) vbits = nz_bits4(vm.x) | (nz_bits4(vm.y) << 4) | (nz_bits4(vm.z) << 8) | (nz_bits4(vm.w) << 12);
        return ((tile << 5) + lane < nv) ? (mine & vbits) : 0u;
    }
};

// Software pipeline: the loads of the warp's NEXT tile are issued before the hits of the current one
// are written, so the dependent read of the `edited` bytes (hit vectors only) overlaps the next
// attribute fetch instead of adding a second DRAM round trip to every step.  The grid is exactly
// the resident blocks (persistent warps, static stride): no partial last wave.
template <int KIND, int ES>
__global__ void __launch_bounds__(BLOCK, ML_THR_VEC_MINB)
threshold_vec_kernel(const void* __restrict__ attr_, const uint8_t* __restrict__ valid, long long n,
                     double lo, double hi, Thr thr, void* __restrict__ data, int esize, uint32_t value,
                     uint8_t* __restrict__ mask, uint8_t* __restrict__ edited, unsigned long long* counter) {
    typedef typename AttrT<KIND>::T T;
    const T* attr = (const T*)attr_;
    long long cnt = 0;
    const int lane = threadIdx.x & 31;
    const long long nv = n >> 4;                                       // whole 16-texel vectors
    const long long ntiles = (nv + 31) >> 5;                           // 512-texel warp tiles
    const long long nwarps = ((long long)gridDim.x * BLOCK) >> 5;
    long long t = ((long long)blockIdx.x * BLOCK + threadIdx.x) >> 5;
    ThrTile<KIND, ES> A, B;
    auto commit = [&](const ThrTile<KIND, ES>& X, long long tile) {
        const unsigned hit16 = X.hits(thr, tile, nv, lane);
        const long long i0 = ((tile << 5) + lane) << 4;
        uint4 ew, mw, dw;
        vec16_load<ES>(data, mask, edited, i0, hit16, ew, mw, dw);
        vec16_commit<ES>(data, value, mask, edited, i0, hit16, ew, mw, dw, cnt);
    };
#if ML_THR_PIPE
    if (t < ntiles) {
        A.load(attr, valid, t, nv, lane);
        while (true) {
            if (t + nwarps < ntiles) B.load(attr, valid, t + nwarps, nv, lane);
            commit(A, t);
            t += nwarps;
            if (t >= ntiles) break;
            if (t + nwarps < ntiles) A.load(attr, valid, t + nwarps, nv, lane);
            commit(B, t);
            t += nwarps;
            if (t >= ntiles) break;
        }
    }
#else
    for (; t < ntiles; t += 2 * nwarps) {          // two tiles in flight per warp, no carry-over between steps
        A.load(attr, valid, t, nv, lane);
        if (t + nwarps < ntiles) B.load(attr, valid, t + nwarps, nv, lane);
        const unsigned ha = A.hits(thr, t, nv, lane);
        const unsigned hb = t + nwarps < ntiles ? B.hits(thr, t + nwarps, nv, lane) : 0u;
        const long long ia = ((t << 5) + lane) << 4, ib = (((t + nwarps) << 5) + lane) << 4;
        uint4 ew[2], mw[2], dw[2];
        vec16_load<ES>(data, mask, edited, ia, ha, ew[0], mw[0], dw[0]);
        vec16_load<ES>(data, mask, edited, ib, hb, ew[1], mw[1], dw[1]);
        vec16_commit<ES>(data, value, mask, edited, ia, ha, ew[0], mw[0], dw[0], cnt);
        vec16_commit<ES>(data, value, mask, edited, ib, hb, ew[1], mw[1], dw[1], cnt);
    }
#endif
    const long long tid = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * BLOCK;
    for (long long i = (nv << 4) + tid; i < n; i += nthreads) {           // < 16 texels of tail
        if (valid && valid[i] == 0) continue;
        const double v = AttrT<KIND>::get(attr[i]);
        if (lo <= v && v <= hi) hit_write(data, esize, value, mask, edited, i, cnt);
    }
    block_count_add(cnt, counter);
}

// Bulk-copy form (default): the attribute plane -- the kernel's read stream -- travels through a
// THB_STAGES x 16 KB shared-memory ring filled by one producer lane per block with cp.async.bulk
// (bulk.cuh), so the HBM pipe stays full while a consumer warp waits for the `edited` bytes of its
// hit vectors (the register forms above alternate between the two round trips and top out near
// 0.6 of the peak with the bench's 19 % coherent hits).  Consumer warps read their tiles from the
// stage lane-interleaved (conflict-free 128-bit LDS) and use the same shuffle transposition and
// 128-bit byte-plane accesses as threshold_vec_kernel.
#ifndef ML_THB_STAGES
#define ML_THB_STAGES 2
#endif
#ifndef ML_THB_CHUNK
#define ML_THB_CHUNK 32768
#endif
#ifndef ML_THB_CW
#define ML_THB_CW 8
#endif
constexpr int THB_STAGES = ML_THB_STAGES;
constexpr int THB_CHUNK = ML_THB_CHUNK;                // attribute bytes per chunk
constexpr int THB_CW = ML_THB_CW;                      // consumer warps
constexpr int THB_THREADS = 32 * (THB_CW + 1);
typedef BulkRing<THB_STAGES, THB_CHUNK> ThrRing;

template <int KIND, int ES, bool HV>
__global__ void __launch_bounds__(THB_THREADS)
threshold_bulk_kernel(const void* __restrict__ attr_, const uint8_t* __restrict__ valid, long long n,
                      double lo, double hi, Thr thr, void* __restrict__ data, int esize, uint32_t value,
                      uint8_t* __restrict__ mask, uint8_t* __restrict__ edited, unsigned long long* counter) {
    typedef typename AttrT<KIND>::T T;
    constexpr int S = (int)sizeof(T);
    constexpr int TILE_BYTES = 512 * S;                     // attribute bytes of one 512-texel warp tile
    constexpr int TPW = THB_CHUNK / TILE_BYTES / THB_CW;    // tiles per consumer warp and chunk (1, 2, 4)
    static_assert(TPW >= 1, "chunk too small for the consumer warps");
    extern __shared__ __align__(128) uint8_t thb_smem[];
    ThrRing& ring = *reinterpret_cast<ThrRing*>(thb_smem);
    const T* attr = (const T*)attr_;
    const long long nv = n >> 4;                            // whole 16-texel vectors
    const long long abytes = nv * 16 * S;                   // their attribute bytes
    const long long nchunks = (abytes + THB_CHUNK - 1) / THB_CHUNK;
    if (threadIdx.x == 0) ring.init(THB_CW);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    long long cnt = 0;
    RingPos<THB_STAGES> pos;
    if (warp == THB_CW) {
        if (lane == 0) {
            const uint64_t policy = l2_policy_evict_first();
            for (long long c = blockIdx.x; c < nchunks; c += gridDim.x, pos.next()) {
                const long long base = c * THB_CHUNK;
                const unsigned bytes = (unsigned)(abytes - base < THB_CHUNK ? abytes - base : THB_CHUNK);
                ring.produce(pos, (const uint8_t*)attr + base, bytes, policy);
            }
        }
    } else {
        for (long long c = blockIdx.x; c < nchunks; c += gridDim.x, pos.next()) {
            const long long base = c * THB_CHUNK;
            const unsigned bytes = (unsigned)(abytes - base < THB_CHUNK ? abytes - base : THB_CHUNK);
            const uint8_t* b = ring.acquire(pos);
            ThrTile<KIND, ES, HV> X[TPW];
            const long long tile0 = base / TILE_BYTES + warp * TPW;        // this warp's first tile of the chunk
#pragma unroll
            for (int j = 0; j < TPW; ++j) {
                const unsigned toff = (unsigned)(warp * TPW + j) * TILE_BYTES;
                X[j].load_smem(b + toff, bytes > toff ? bytes - toff : 0u, valid, tile0 + j, nv, lane);
            }
            ring.release(pos);
            unsigned hit16[TPW];
            uint4 ew[TPW], mw[TPW], dw[TPW];
#pragma unroll
            for (int j = 0; j < TPW; ++j) hit16[j] = X[j].hits(thr, tile0 + j, nv, lane);
#pragma unroll
            for (int j = 0; j < TPW; ++j)
                vec16_load<ES>(data, mask, edited, (((tile0 + j) << 5) + lane) << 4, hit16[j], ew[j], mw[j], dw[j]);
#pragma unroll
            for (int j = 0; j < TPW; ++j)
                vec16_commit<ES>(data, value, mask, edited, (((tile0 + j) << 5) + lane) << 4, hit16[j], ew[j], mw[j], dw[j], cnt);
        }
        if (blockIdx.x == 0) {
            for (long long i = (nv << 4) + threadIdx.x; i < n; i += 32 * THB_CW) {       // < 16 texels of tail
                if (valid && valid[i] == 0) continue;
                const double v = AttrT<KIND>::get(attr[i]);
                if (lo <= v && v <= hi) hit_write(data, esize, value, mask, edited, i, cnt);
            }
        }
    }
    block_count_add(cnt, counter);
}

// ---------------------------------------------------------------------------------------------
// thresholds rounded inward once, in every attribute domain; false for an empty or NaN interval
inline bool make_thr(double lo, double hi, Thr& thr) {
    if (!(lo <= hi)) return false;
    thr.lo_f = (float)lo; if ((double)thr.lo_f < lo) thr.lo_f = nextafterf(thr.lo_f, INFINITY);
    thr.hi_f = (float)hi; if ((double)thr.hi_f > hi) thr.hi_f = nextafterf(thr.hi_f, -INFINITY);
    const double big = 9.2e18;
    thr.lo_i = lo <= -big ? LLONG_MIN : (lo >= big ? LLONG_MAX : (long long)ceil(lo));
    thr.hi_i = hi >= big ? LLONG_MAX : (hi <= -big ? LLONG_MIN : (long long)floor(hi));
    return true;
}

inline unsigned stream_grid(long long items_per_thread_iter, long long n_items) {
    long long blocks = (n_items + (long long)BLOCK * items_per_thread_iter - 1) / ((long long)BLOCK * items_per_thread_iter);
    const long long cap = (long long)ml_sm_count() * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (unsigned)blocks;
}

inline bool aligned(const void* p, size_t a) { return ((uintptr_t)p % a) == 0; }
inline bool planes_aligned(const void* d, const void* m, const void* e) { return aligned(d, 16) && aligned(m, 16) && aligned(e, 16); }

template <int KIND>
int launch_threshold(const void* attr, const uint8_t* valid, long long n, double lo, double hi,
                     void* data, int esize, uint32_t value, uint8_t* mask, uint8_t* edited,
                     unsigned long long* counter, cudaStream_t st) {
    typedef typename AttrT<KIND>::T T;
    const bool vec = aligned(attr, sizeof(T) * 4) && (!valid || aligned(valid, 4)) && planes_aligned(data, mask, edited);
    const unsigned grid = stream_grid(4 * TU, n);
    Thr thr;
    if (!make_thr(lo, hi, thr)) return ML_OK;  // empty or NaN interval: nothing can hit
    static const bool quad_form = getenv("ML_THR_QUAD_STREAM") != nullptr;              // the round-1 kernel, kept for comparison
    if (vec && !quad_form && aligned(attr, 16) && (!valid || aligned(valid, 16)) && n >= 512) {
        static const bool reg_form = getenv("ML_THR_REGISTER_STREAM") != nullptr;     // threshold_vec_kernel, kept for comparison
        if (!reg_form && n >= 4 * THB_CHUNK) {
            static int per_sm_b[6] = {0, 0, 0, 0, 0, 0};
            const int kb = (esize == 1 ? 0 : (esize == 2 ? 1 : 2)) + (valid ? 3 : 0);
            const void* fb = valid ? (esize == 1 ? (const void*)threshold_bulk_kernel<KIND, 1, true>
                                   : (esize == 2 ? (const void*)threshold_bulk_kernel<KIND, 2, true> : (const void*)threshold_bulk_kernel<KIND, 4, true>))
                                   : (esize == 1 ? (const void*)threshold_bulk_kernel<KIND, 1, false>
                                   : (esize == 2 ? (const void*)threshold_bulk_kernel<KIND, 2, false> : (const void*)threshold_bulk_kernel<KIND, 4, false>));
            if (!per_sm_b[kb]) {
                ML_CUDA(cudaFuncSetAttribute(fb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ThrRing)));
                int nb = 0;
                ML_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fb, THB_THREADS, sizeof(ThrRing)));
                per_sm_b[kb] = nb > 0 ? nb : 1;
            }
            const long long nchunks = ((n >> 4) * 16 * (long long)sizeof(T) + THB_CHUNK - 1) / THB_CHUNK;
            long long gb = (long long)ml_sm_count() * per_sm_b[kb];
            if (gb > nchunks) gb = nchunks;
            void* kargs[] = {(void*)&attr, (void*)&valid, (void*)&n, (void*)&lo, (void*)&hi, (void*)&thr, (void*)&data, (void*)&esize,
                             (void*)&value, (void*)&mask, (void*)&edited, (void*)&counter};
            ML_CUDA(cudaLaunchKernel(fb, dim3((unsigned)gb), dim3(THB_THREADS), kargs, sizeof(ThrRing), st));
            return ML_OK;
        }
        static int per_sm[3] = {0, 0, 0};                             // resident blocks per SM of each instantiation
        const int k = esize == 1 ? 0 : (esize == 2 ? 1 : 2);
        const void* fn = esize == 1 ? (const void*)threshold_vec_kernel<KIND, 1>
                       : (esize == 2 ? (const void*)threshold_vec_kernel<KIND, 2> : (const void*)threshold_vec_kernel<KIND, 4>);
        if (!per_sm[k]) {
            int nb = 0;
            ML_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, BLOCK, 0));
            per_sm[k] = nb > 0 ? nb : 1;
        }
        long long g16 = (long long)ml_sm_count() * per_sm[k] * ML_THR_WAVES;
        const long long need = ((n >> 9) + BLOCK / 32) / (BLOCK / 32);       // one warp tile per warp at least
        if (g16 > need) g16 = need;
        if (g16 < 1) g16 = 1;
#define ML_LAUNCH_THRV(ES) threshold_vec_kernel<KIND, ES><<<(unsigned)g16, BLOCK, 0, st>>>(attr, valid, n, lo, hi, thr, data, esize, value, mask, edited, counter)
        if (esize == 1) ML_LAUNCH_THRV(1); else if (esize == 2) ML_LAUNCH_THRV(2); else ML_LAUNCH_THRV(4);
#undef ML_LAUNCH_THRV
        ML_CUDA(cudaGetLastError());
        return ML_OK;
    }
#define ML_LAUNCH_THR(ES) threshold_kernel<KIND, ES><<<grid, BLOCK, 0, st>>>(attr, valid, n, lo, hi, thr, data, esize, value, mask, edited, counter)
    if (!vec) ML_LAUNCH_THR(0);
    else if (esize == 1) ML_LAUNCH_THR(1);
    else if (esize == 2) ML_LAUNCH_THR(2);
    else ML_LAUNCH_THR(4);
#undef ML_LAUNCH_THR
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

}  // namespace

extern "C" {

int ml_select_sphere(const float* pos, int64_t pos_stride, int64_t n,
                     double cx, double cy, double cz, double radius,
                     void* data, int esize, uint32_t value_bits, uint8_t* mask, uint8_t* edited,
                     uint64_t* count, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (esize != 1 && esize != 2 && esize != 4) return ml_fail(ML_ERR_ARG, "esize must be 1, 2 or 4");
    if (n <= 0) return ML_OK;
    const float *px = pos, *py = pos + pos_stride, *pz = pos + 2 * pos_stride;
    const double r2 = radius * radius;      // host IEEE multiply == the oracle's r*r
    const bool vec = aligned(px, 16) && aligned(py, 16) && aligned(pz, 16) && planes_aligned(data, mask, edited);
    const unsigned grid = stream_grid(4 * UNROLL, n);
    unsigned long long* c = (unsigned long long*)count;
#define ML_LAUNCH_SPH(ES) sphere_kernel<ES><<<grid, BLOCK, 0, st>>>(px, py, pz, n, cx, cy, cz, r2, data, esize, value_bits, mask, edited, c)
    if (!vec) ML_LAUNCH_SPH(0);
    else if (esize == 1) ML_LAUNCH_SPH(1);
    else if (esize == 2) ML_LAUNCH_SPH(2);
    else ML_LAUNCH_SPH(4);
#undef ML_LAUNCH_SPH
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int ml_select_sphere_batch(const float* pos, int64_t pos_stride, int64_t n,
                           const double* strokes, const int32_t* layer_of,
                           const uint32_t* value_bits, int64_t K,
                           void* const* data, uint8_t* const* mask, uint8_t* const* edited,
                           int64_t L, int esize, uint64_t* counts, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (esize != 1 && esize != 2 && esize != 4) return ml_fail(ML_ERR_ARG, "esize must be 1, 2 or 4");
    if (n <= 0 || K <= 0) return ML_OK;
    const float *px = pos, *py = pos + pos_stride, *pz = pos + 2 * pos_stride;
    if (!(aligned(px, 16) && aligned(py, 16) && aligned(pz, 16)) || (n & 3))
        return ml_fail(ML_ERR_ARG, "batched sphere brush needs 16-byte aligned planes and n % 4 == 0");
    BatchArgs a{px, py, pz, n, strokes, layer_of, value_bits, K, data, mask, edited, L,
                (unsigned long long*)counts};
    const long long nunits = ((n >> 2) + 127) >> 7;
    long long blocks = (nunits + BLOCK / 32 - 1) / (BLOCK / 32);
    const long long cap = (long long)ml_sm_count() * 16;
    if (blocks > cap) blocks = cap;
    if (esize == 1) sphere_batch_kernel<1><<<(unsigned)blocks, BLOCK, 0, st>>>(a);
    else if (esize == 2) sphere_batch_kernel<2><<<(unsigned)blocks, BLOCK, 0, st>>>(a);
    else sphere_batch_kernel<4><<<(unsigned)blocks, BLOCK, 0, st>>>(a);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int64_t ml_tile_count(int64_t width, int64_t rows) {
    if (width <= 0 || rows <= 0 || (width & ((1 << ST_W_SHIFT) - 1)) != 0) return 0;
    return tile_grid(width, rows).ntiles;
}

size_t ml_tile_workspace_bytes(int64_t width, int64_t rows) {
    const long long nt = ml_tile_count(width, rows);
    return 16 + (size_t)(tile_bitmap_words(nt) + nt) * sizeof(uint32_t);
}

int ml_surface_tile_boxes(const float* pos, int64_t pos_stride, int64_t width, int64_t rows,
                          float* boxes, void* stream) {
    const long long ntiles = ml_tile_count(width, rows);
    if (ntiles == 0) return ml_fail(ML_ERR_ARG, "tile boxes need width % 128 == 0");
    const float *px = pos, *py = pos + pos_stride, *pz = pos + 2 * pos_stride;
    if (!(aligned(px, 16) && aligned(py, 16) && aligned(pz, 16) && aligned(boxes, 16)))
        return ml_fail(ML_ERR_ARG, "tile boxes need 16-byte aligned planes");
    long long blocks = (ntiles + BLOCK / 32 - 1) / (BLOCK / 32);
    const long long cap = (long long)ml_sm_count() * 16;
    if (blocks > cap) blocks = cap;
    tile_box_kernel<<<(unsigned)blocks, BLOCK, 0, (cudaStream_t)stream>>>(px, py, pz, tile_grid(width, rows), (float4*)boxes);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

static int tiles_prepare(int64_t width, int64_t rows, const float* boxes, void* workspace, size_t workspace_bytes,
                         const double* strokes, long long K, double cx, double cy, double cz, double cr,
                         TileGrid& g, TileList& list, cudaStream_t st) {
    if (ml_tile_count(width, rows) == 0) return ml_fail(ML_ERR_ARG, "culled brushes need width % 128 == 0");
    if (boxes == nullptr || !aligned(boxes, 16)) return ml_fail(ML_ERR_ARG, "culled brushes need the 16-byte aligned tile boxes");
    if (workspace == nullptr || workspace_bytes < ml_tile_workspace_bytes(width, rows) || !aligned(workspace, 8))
        return ml_fail(ML_ERR_ARG, "culled brushes need ml_tile_workspace_bytes() of 8-byte aligned scratch");
    g = tile_grid(width, rows);
    list.count = (unsigned long long*)workspace;
    list.bits = (uint32_t*)(list.count + 2);
    list.tiles = list.bits + tile_bitmap_words(g.ntiles);
    ML_CUDA(cudaMemsetAsync(workspace, 0, 16 + (size_t)tile_bitmap_words(g.ntiles) * 4, st));      // count + bitmap
    long long chunks = strokes ? (K + KC - 1) / KC : 1;
    if (chunks > 1024) chunks = 1024;                                 // the kernel strides over the rest
    const dim3 grid((unsigned)((g.ntiles + BLOCK - 1) / BLOCK), (unsigned)chunks);
    tile_classify_kernel<<<grid, BLOCK, 0, st>>>((const float4*)boxes, g.ntiles, strokes, K, cx, cy, cz, cr, list);
    return ML_OK;
}

int ml_select_sphere_tiles(const float* pos, int64_t pos_stride, int64_t width, int64_t rows,
                           const float* boxes, void* workspace, size_t workspace_bytes,
                           double cx, double cy, double cz, double radius,
                           void* data, int esize, uint32_t value_bits, uint8_t* mask, uint8_t* edited,
                           uint64_t* count, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (esize != 1 && esize != 2 && esize != 4) return ml_fail(ML_ERR_ARG, "esize must be 1, 2 or 4");
    if (width <= 0 || rows <= 0) return ML_OK;
    const float *px = pos, *py = pos + pos_stride, *pz = pos + 2 * pos_stride;
    if (!(aligned(px, 16) && aligned(py, 16) && aligned(pz, 16) && planes_aligned(data, mask, edited)))
        return ml_fail(ML_ERR_ARG, "culled sphere brush needs 16-byte aligned planes");
    TileGrid g; TileList list;
    const int rc = tiles_prepare(width, rows, boxes, workspace, workspace_bytes, nullptr, 1, cx, cy, cz, radius, g, list, st);
    if (rc != ML_OK) return rc;
    const double r2 = radius * radius;      // host IEEE multiply == the oracle's r*r
    const unsigned grid = (unsigned)(ml_sm_count() * 8);
    unsigned long long* c = (unsigned long long*)count;
    if (esize == 1) sphere_tiles_kernel<1><<<grid, BLOCK, 0, st>>>(px, py, pz, g, list, cx, cy, cz, r2, data, value_bits, mask, edited, c);
    else if (esize == 2) sphere_tiles_kernel<2><<<grid, BLOCK, 0, st>>>(px, py, pz, g, list, cx, cy, cz, r2, data, value_bits, mask, edited, c);
    else sphere_tiles_kernel<4><<<grid, BLOCK, 0, st>>>(px, py, pz, g, list, cx, cy, cz, r2, data, value_bits, mask, edited, c);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int ml_select_sphere_batch_tiles(const float* pos, int64_t pos_stride, int64_t width, int64_t rows,
                                 const float* boxes, void* workspace, size_t workspace_bytes,
                                 const double* strokes, const int32_t* layer_of,
                                 const uint32_t* value_bits, int64_t K,
                                 void* const* data, uint8_t* const* mask, uint8_t* const* edited,
                                 int64_t L, int esize, uint64_t* counts, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (esize != 1 && esize != 2 && esize != 4) return ml_fail(ML_ERR_ARG, "esize must be 1, 2 or 4");
    if (width <= 0 || rows <= 0 || K <= 0) return ML_OK;
    const float *px = pos, *py = pos + pos_stride, *pz = pos + 2 * pos_stride;
    if (!(aligned(px, 16) && aligned(py, 16) && aligned(pz, 16)))
        return ml_fail(ML_ERR_ARG, "batched sphere brush needs 16-byte aligned planes");
    TileGrid g; TileList list;
    const int rc = tiles_prepare(width, rows, boxes, workspace, workspace_bytes, strokes, K, 0.0, 0.0, 0.0, 0.0, g, list, st);
    if (rc != ML_OK) return rc;
    BatchArgs a{px, py, pz, (long long)width * rows, strokes, layer_of, value_bits, K, data, mask, edited, L,
                (unsigned long long*)counts};
    const unsigned grid = (unsigned)(ml_sm_count() * 8);
    if (esize == 1) sphere_batch_tiles_kernel<1><<<grid, BLOCK, 0, st>>>(a, g, (const float4*)boxes, list);
    else if (esize == 2) sphere_batch_tiles_kernel<2><<<grid, BLOCK, 0, st>>>(a, g, (const float4*)boxes, list);
    else sphere_batch_tiles_kernel<4><<<grid, BLOCK, 0, st>>>(a, g, (const float4*)boxes, list);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int ml_plane_tile_range(const float* attr, int64_t width, int64_t rows, float* ranges, void* stream) {
    const long long ntiles = ml_tile_count(width, rows);
    if (ntiles == 0) return ml_fail(ML_ERR_ARG, "tile ranges need width % 128 == 0");
    if (!aligned(attr, 16) || !aligned(ranges, 8)) return ml_fail(ML_ERR_ARG, "tile ranges need a 16-byte aligned plane");
    long long blocks = (ntiles + BLOCK / 32 - 1) / (BLOCK / 32);
    const long long cap = (long long)ml_sm_count() * 16;
    if (blocks > cap) blocks = cap;
    tile_range_kernel<<<(unsigned)blocks, BLOCK, 0, (cudaStream_t)stream>>>(attr, tile_grid(width, rows), (float2*)ranges);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int ml_select_threshold_tiles(const float* attr, const uint8_t* valid, int64_t width, int64_t rows,
                              const float* ranges, void* workspace, size_t workspace_bytes,
                              double lo, double hi, void* data, int esize, uint32_t value_bits,
                              uint8_t* mask, uint8_t* edited, uint64_t* count, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (esize != 1 && esize != 2 && esize != 4) return ml_fail(ML_ERR_ARG, "esize must be 1, 2 or 4");
    if (width <= 0 || rows <= 0) return ML_OK;
    if (ml_tile_count(width, rows) == 0) return ml_fail(ML_ERR_ARG, "culled threshold needs width % 128 == 0");
    if (ranges == nullptr || !aligned(ranges, 8) || !aligned(attr, 16) || (valid && !aligned(valid, 4)) ||
        !planes_aligned(data, mask, edited))
        return ml_fail(ML_ERR_ARG, "culled threshold needs the tile ranges and 16-byte aligned planes");
    if (workspace == nullptr || workspace_bytes < ml_tile_workspace_bytes(width, rows) || !aligned(workspace, 8))
        return ml_fail(ML_ERR_ARG, "culled threshold needs ml_tile_workspace_bytes() of 8-byte aligned scratch");
    Thr thr;
    if (!make_thr(lo, hi, thr)) return ML_OK;
    const TileGrid g = tile_grid(width, rows);
    TileList list;
    list.count = (unsigned long long*)workspace;
    list.bits = (uint32_t*)(list.count + 2);
    list.tiles = list.bits + tile_bitmap_words(g.ntiles);
    ML_CUDA(cudaMemsetAsync(workspace, 0, 16, st));
    range_classify_kernel<<<(unsigned)((g.ntiles + BLOCK - 1) / BLOCK), BLOCK, 0, st>>>((const float2*)ranges, g.ntiles,
                                                                                       thr.lo_f, thr.hi_f, list);
    const unsigned grid = (unsigned)(ml_sm_count() * 16);
    unsigned long long* c = (unsigned long long*)count;
    static const bool quad_form = getenv("ML_THR_QUAD_STREAM") != nullptr;              // the round-1 tile walk, kept for comparison
    if (!quad_form && (!valid || aligned(valid, 16))) {
#define ML_LAUNCH_TTV(ES) do { \
        if (valid) threshold_tiles_vec_kernel<ES, true><<<grid, BLOCK, 0, st>>>(attr, valid, g, list, thr, data, value_bits, mask, edited, c); \
        else threshold_tiles_vec_kernel<ES, false><<<grid, BLOCK, 0, st>>>(attr, valid, g, list, thr, data, value_bits, mask, edited, c); } while (0)
        if (esize == 1) ML_LAUNCH_TTV(1);
        else if (esize == 2) ML_LAUNCH_TTV(2);
        else ML_LAUNCH_TTV(4);
#undef ML_LAUNCH_TTV
    }
    else if (esize == 1) threshold_tiles_kernel<1><<<grid, BLOCK, 0, st>>>(attr, valid, g, list, thr, data, value_bits, mask, edited, c);
    else if (esize == 2) threshold_tiles_kernel<2><<<grid, BLOCK, 0, st>>>(attr, valid, g, list, thr, data, value_bits, mask, edited, c);
    else threshold_tiles_kernel<4><<<grid, BLOCK, 0, st>>>(attr, valid, g, list, thr, data, value_bits, mask, edited, c);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int ml_select_threshold(const void* attr, int attr_kind, const uint8_t* valid, int64_t n,
                        double lo, double hi, void* data, int esize, uint32_t value_bits,
                        uint8_t* mask, uint8_t* edited, uint64_t* count, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (esize != 1 && esize != 2 && esize != 4) return ml_fail(ML_ERR_ARG, "esize must be 1, 2 or 4");
    if (n <= 0) return ML_OK;
    unsigned long long* c = (unsigned long long*)count;
    switch (attr_kind) {
    case ML_U8:  return launch_threshold<ML_U8>(attr, valid, n, lo, hi, data, esize, value_bits, mask, edited, c, st);
    case ML_I8:  return launch_threshold<ML_I8>(attr, valid, n, lo, hi, data, esize, value_bits, mask, edited, c, st);
    case ML_I16: return launch_threshold<ML_I16>(attr, valid, n, lo, hi, data, esize, value_bits, mask, edited, c, st);
    case ML_I32: return launch_threshold<ML_I32>(attr, valid, n, lo, hi, data, esize, value_bits, mask, edited, c, st);
    case ML_U32: return launch_threshold<ML_U32>(attr, valid, n, lo, hi, data, esize, value_bits, mask, edited, c, st);
    case ML_F16: return launch_threshold<ML_F16>(attr, valid, n, lo, hi, data, esize, value_bits, mask, edited, c, st);
    case ML_FLOAT32: return launch_threshold<ML_FLOAT32>(attr, valid, n, lo, hi, data, esize, value_bits, mask, edited, c, st);
    }
    return ml_fail(ML_ERR_ARG, "unknown attribute kind");
}

}  // extern "C"
