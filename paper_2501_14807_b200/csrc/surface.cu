// Per-texel kernels that run over the cached triangle-id map:
//   ml_surface_resolve : position / normal / area map (north star (1); oracle ext_surface_map)
//   ml_tea_texels      : the paper's projective brush (TEA) evaluated per texel for the owner
//                        triangle -- bit-identical to the per-triangle reference loop
//                        (KN:135-203) when uv islands do not overlap (SURVEY.md 8 note N1).
// One thread per texel, consecutive threads on consecutive texels of a row: the 4-byte id read
// is a coalesced stream; the triangle records are gathers that hit L1/L2 because neighbouring
// texels share their owner.
#include <stdlib.h>
#include "common.cuh"
#include "bulk.cuh"
#include "meshlayers_b200.h"
#include "internal.h"

namespace {

constexpr int BLOCK = 256;

// Texel (x, y) of flat slab index i; 32-bit division when the slab is small enough.
ML_DEV void texel_xy(long long i, long long width, long long row0, bool small, int& x, int& y) {
    if (small) {
        const unsigned yy = (unsigned)i / (unsigned)width;
        x = (int)((unsigned)i - yy * (unsigned)width); y = (int)(row0 + yy);
    } else {
        const long long yy = i / width;
        x = (int)(i - yy * width); y = (int)(row0 + yy);
    }
}

// Per-triangle record of the resolve pass (208 bytes = 13 x 16, written once per build by
// tri_prepare_kernel): the CCW-normalised uv vertices (KN:32-41), the texel area of the triangle
// (3D area / uv area, constant over the triangle) and the position / normal attributes widened to
// float64 in CCW vertex order (KN:40 swaps the attributes with the vertices).  The per-texel kernel
// fetches it with thirteen independent 128-bit loads issued back to back, and neither re-derives
// the winding nor repeats the cross product, square root and division for every texel.
struct __align__(16) TriRec {
    double x0, y0, x1, y1, x2, y2;
    float area;
    uint32_t flags;                   // bit 0 valid, bit 1 vertices 1 and 2 were exchanged
    double pad;
    double p[9];                      // p0.xyz, p1.xyz, p2.xyz (CCW order)
    double nrm[9];
};
static_assert(sizeof(TriRec) == 208, "TriRec is thirteen 16-byte words");

template <typename T>
__global__ void __launch_bounds__(BLOCK)
tri_prepare_kernel(const T* __restrict__ tri_xy, const T* __restrict__ tri_pos, const T* __restrict__ tri_nrm,
                   long long ntri, TriRec* __restrict__ recs, const int* __restrict__ slab_list,
                   const unsigned long long* __restrict__ slab_count) {
    // row slabs: only the triangles of the slab's list can own a texel of the slab, only their records are needed
    const long long k = (long long)blockIdx.x * BLOCK + threadIdx.x;
    if (k >= (slab_list ? (long long)*slab_count : ntri)) return;
    const long long t = slab_list ? (long long)slab_list[k] : k;
    TriSetup s;
    TriRec& r = recs[t];
    if (!tri_load_ccw(tri_xy + 6 * t, s)) {       // degenerate / non-finite: never owns a texel
        r.flags = 0u;
        return;
    }
    r.x0 = s.x0; r.y0 = s.y0; r.x1 = s.x1; r.y1 = s.y1; r.x2 = s.x2; r.y2 = s.y2;
    r.flags = 1u | (s.swapped ? 2u : 0u);
    r.pad = 0.0;
    const int i1 = s.swapped ? 6 : 3, i2 = s.swapped ? 3 : 6;
    const T* P = tri_pos + 9 * t;
    const T* N = tri_nrm + 9 * t;
    double p0[3], p1[3], p2[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        p0[c] = (double)P[c]; p1[c] = (double)P[i1 + c]; p2[c] = (double)P[i2 + c];
        r.p[c] = p0[c]; r.p[3 + c] = p1[c]; r.p[6 + c] = p2[c];
        r.nrm[c] = (double)N[c]; r.nrm[3 + c] = (double)N[i1 + c]; r.nrm[6 + c] = (double)N[i2 + c];
    }
    const double ux = xsub(p1[0], p0[0]), uy = xsub(p1[1], p0[1]), uz = xsub(p1[2], p0[2]);
    const double vx = xsub(p2[0], p0[0]), vy = xsub(p2[1], p0[1]), vz = xsub(p2[2], p0[2]);
    const double crx = xsub(xmul(uy, vz), xmul(uz, vy));
    const double cry = xsub(xmul(uz, vx), xmul(ux, vz));
    const double crz = xsub(xmul(ux, vy), xmul(uy, vx));
    const double a3 = xmul(__dsqrt_rn(xadd(xadd(xmul(crx, crx), xmul(cry, cry)), xmul(crz, crz))), 0.5);
    // |area2| of the CCW-normalised triangle: swapping two vertices negates KN:35 exactly
    const double area2 = xsub(xmul(s.cx, xsub(s.y2, s.y0)), xmul(s.cy, xsub(s.x2, s.x0)));
    const double a2 = xmul(fabs(area2), 0.5);
    r.area = (float)xdiv(a3, a2);
}

// One thread per texel, consecutive lanes on consecutive texels: id reads and the seven plane
// stores are coalesced streams; the record gathers hit L1 because neighbours share owners.  The
// next iteration's id is fetched before this iteration's arithmetic, and the whole record is loaded
// before the first division (whose slow-path call would otherwise fence the remaining loads).
#ifndef ML_RESOLVE_MINB
#define ML_RESOLVE_MINB 4
#endif
template <bool SMALL>
__global__ void __launch_bounds__(BLOCK, ML_RESOLVE_MINB)
resolve_kernel(const TriRec* __restrict__ recs, long long width, long long row0, long long n,
               const int* __restrict__ tri_id, float* __restrict__ pos, float* __restrict__ nrm,
               float* __restrict__ area, unsigned long long* covered) {
    long long cnt = 0;
    const long long stride = (long long)gridDim.x * BLOCK;
    long long i = (long long)blockIdx.x * BLOCK + threadIdx.x;
    int t = i < n ? (int)ld_stream((const uint32_t*)tri_id + i) : -1;
    for (; i < n; i += stride) {
        const int tcur = t;
        if (i + stride < n) t = (int)ld_stream((const uint32_t*)tri_id + i + stride);
        if (tcur < 0) {
            const float qnan = __int_as_float(0x7fc00000);
            pos[i] = qnan; pos[n + i] = qnan; pos[2 * n + i] = qnan;
            nrm[i] = 0.f; nrm[n + i] = 0.f; nrm[2 * n + i] = 0.f;
            area[i] = 0.f;
            continue;
        }
        ++cnt;
        // The 208-byte record is consumed in three rounds (uv vertices -> barycentrics, positions,
        // normals), each fetched right before its arithmetic: the kernel then fits 64 registers and
        // twice as many warps hide the float64 latency (the record's lines are in L1 after round 1).
        const double2* rp = (const double2*)(recs + tcur);
        const double2 v0 = __ldg(rp), v1 = __ldg(rp + 1), v2 = __ldg(rp + 2), af = __ldg(rp + 3);
        int x, y;
        texel_xy(i, width, row0, SMALL, x, y);
        const double cx = xadd((double)x, 0.5), cy = xadd((double)y, 0.5);                            // KN:60, 63
        const double e0 = xsub(xmul(xsub(v2.x, v1.x), xsub(cy, v1.y)), xmul(xsub(v2.y, v1.y), xsub(cx, v1.x)));   // KN:72
        const double e1 = xsub(xmul(xsub(v0.x, v2.x), xsub(cy, v2.y)), xmul(xsub(v0.y, v2.y), xsub(cx, v2.x)));   // KN:73
        const double e2 = xsub(xmul(xsub(v1.x, v0.x), xsub(cy, v0.y)), xmul(xsub(v1.y, v0.y), xsub(cx, v0.x)));   // KN:74
        area[i] = __uint_as_float((uint32_t)__double_as_longlong(af.x));      // low word of bytes 48..55 = TriRec::area
        const double esum = xadd(xadd(e0, e1), e2);
        const double l0 = xdiv(e0, esum), l1 = xdiv(e1, esum), l2 = xdiv(e2, esum);
        {   // positions: record words 4..8 = p0.xyz, p1.xyz, p2.xyz (+ nrm[0] in w8.y)
            const double2 w4 = __ldg(rp + 4), w5 = __ldg(rp + 5), w6 = __ldg(rp + 6), w7 = __ldg(rp + 7), w8 = __ldg(rp + 8);
            pos[i] = (float)xadd(xadd(xmul(l0, w4.x), xmul(l1, w5.y)), xmul(l2, w7.x));
            pos[n + i] = (float)xadd(xadd(xmul(l0, w4.y), xmul(l1, w6.x)), xmul(l2, w7.y));
            pos[2 * n + i] = (float)xadd(xadd(xmul(l0, w5.x), xmul(l1, w6.y)), xmul(l2, w8.x));
        }
        // normals: record words 8.y .. 12 = n0.xyz, n1.xyz, n2.xyz
        const double2 w8 = __ldg(rp + 8), w9 = __ldg(rp + 9), w10 = __ldg(rp + 10), w11 = __ldg(rp + 11), w12 = __ldg(rp + 12);
        const double nx = xadd(xadd(xmul(l0, w8.y), xmul(l1, w10.x)), xmul(l2, w11.y));
        const double ny = xadd(xadd(xmul(l0, w9.x), xmul(l1, w10.y)), xmul(l2, w12.x));
        const double nz = xadd(xadd(xmul(l0, w9.y), xmul(l1, w11.x)), xmul(l2, w12.y));
        const double len = __dsqrt_rn(xadd(xadd(xmul(nx, nx), xmul(ny, ny)), xmul(nz, nz)));
        const bool ok = len > 0.0;
        nrm[i] = ok ? (float)xdiv(nx, len) : 0.f;
        nrm[n + i] = ok ? (float)xdiv(ny, len) : 0.f;
        nrm[2 * n + i] = ok ? (float)xdiv(nz, len) : 0.f;
    }
    block_count_add(cnt, covered);
}

// ---------------------------------------------------------------------------------------------
// Per-stroke triangle classification.  flags[t] = 0 only when NO texel of triangle t can pass the
// TEA filters, decided from the three vertices alone:
//   * all w_i <= 0: every fragment has wc = (l0*w0 + l1*w1) + l2*w2 <= 0 (l_i >= 0 for covered
//     texels, products and sums of non-positive terms stay non-positive under rounding) -> KN:174;
//   * all w_i > 0: xn = xc/wc is a convex combination of the vertex ratios x_i/w_i (weights
//     l_i*w_i >= 0) up to a rounding error bounded by ~8u*(1 + max|x_i| / min w_i).  If the tool
//     coordinate s = sfx*xn + bx (KN:187) of all three vertices lies on one side of [0,1] by more
//     than delta = 1e-9*(|sfx|*(1 + max|x_i|/min w_i) + |bx| + 1)  (>= 10^6 x the rounding bound)
//     the closed test KN:189 fails for every fragment; likewise for t and for the window test
//     KN:181 (xn outside [-1,1]).
// Anything else (mixed signs of w, NaNs) keeps flag 1.  The texel kernel skips flag-0 triangles,
// which removes the float64 work for everything outside the tool footprint without changing a bit.
// footprint tiles: 128 texels (one warp-wide 128-bit load) x 8 rows
constexpr int TILE_W_SHIFT = 7, TILE_H_SHIFT = 3;
// A tile buffer (ml_tea_tile_words 32-bit words) = [bitmap: tile_bitmap_words][count: u64][list:
// ntiles u32].  The classification pass appends a tile to the list the first time it marks it, so
// the texel pass walks a compact list (one warp per listed tile) instead of every tile of the slab.
__host__ __device__ inline long long tile_bitmap_words(long long ntiles) { return ((ntiles + 63) / 64) * 2; }
struct TileBuf {
    uint32_t* bits; unsigned long long* count; uint32_t* list;
    __host__ __device__ TileBuf(uint32_t* base, long long ntiles)
        : bits(base), count((unsigned long long*)(base + (base ? tile_bitmap_words(ntiles) : 0))),
          list(base + (base ? tile_bitmap_words(ntiles) + 2 : 0)) {}
};

// Footprint tiles (TILE_W x TILE_H texels): every texel a flagged triangle can own lies in its raster
// bbox (the same tri_bbox the rasteriser used), so the marked tiles cover every texel this stroke can
// touch.  A tile is appended to the buffer's list by whoever marks it first.
template <typename T>
ML_DEV void mark_tiles(const T* __restrict__ xy, long long width, long long height, long long row0, long long rows,
                       uint32_t* __restrict__ tile_bits) {
    TriSetup s;
    if (!tri_load_ccw(xy, s) || !tri_bbox(s, width, height, row0, rows)) return;
    const int segs = (int)(width >> TILE_W_SHIFT);
    const TileBuf tb(tile_bits, (long long)segs * ((rows + (1 << TILE_H_SHIFT) - 1) >> TILE_H_SHIFT));
    for (int ty = (int)(s.iy0 - row0) >> TILE_H_SHIFT; ty <= (int)(s.iy1 - row0) >> TILE_H_SHIFT; ++ty)
        for (int tx = s.ix0 >> TILE_W_SHIFT; tx <= s.ix1 >> TILE_W_SHIFT; ++tx) {
            const int tile = ty * segs + tx;
            const uint32_t bit = 1u << (tile & 31);
            if (ld_volatile_u32(tb.bits + (tile >> 5)) & bit) continue;        // already marked
            if (!(atomicOr(tb.bits + (tile >> 5), bit) & bit)) tb.list[atomicAdd(tb.count, 1ull)] = (uint32_t)tile;
        }
}

template <typename T>
__global__ void __launch_bounds__(BLOCK)
tea_classify_kernel(const T* __restrict__ tri_clip, long long ntri, TeaParams p, uint32_t* __restrict__ bits,
                    const T* __restrict__ tri_xy, long long width, long long height, long long row0, long long rows,
                    uint32_t* __restrict__ tile_bits) {
    // output: a BITMAP (bit t&31 of word t>>5), 125 KB per million triangles, so the texel kernel
    // can keep it in shared memory
    const long long t = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const bool live = t < ntri;
    const T* c = tri_clip + 12 * (live ? t : 0);
    double x[3], y[3], w[3];
#pragma unroll
    for (int v = 0; v < 3; ++v) { x[v] = (double)c[4 * v]; y[v] = (double)c[4 * v + 1]; w[v] = (double)c[4 * v + 3]; }
    const int npos = (w[0] > 0.0) + (w[1] > 0.0) + (w[2] > 0.0);
    const int nnonpos = (w[0] <= 0.0) + (w[1] <= 0.0) + (w[2] <= 0.0);
    uint8_t keep = 1;
    if (nnonpos == 3) keep = 0;
    else if (npos == 3) {
        const double wmin = fmin(fmin(w[0], w[1]), w[2]);
        const double ax = fmax(fmax(fabs(x[0]), fabs(x[1])), fabs(x[2])) / wmin;
        const double ay = fmax(fmax(fabs(y[0]), fabs(y[1])), fabs(y[2])) / wmin;
        const double xn0 = x[0] / w[0], xn1 = x[1] / w[1], xn2 = x[2] / w[2];
        const double yn0 = y[0] / w[0], yn1 = y[1] / w[1], yn2 = y[2] / w[2];
        const double xlo = fmin(fmin(xn0, xn1), xn2), xhi = fmax(fmax(xn0, xn1), xn2);
        const double ylo = fmin(fmin(yn0, yn1), yn2), yhi = fmax(fmax(yn0, yn1), yn2);
        const double dxn = 1e-9 * (1.0 + ax), dyn = 1e-9 * (1.0 + ay);
        // tool test: s = sfx*xn + bx over [xlo, xhi] (sfx may be negative)
        const double s0 = p.sfx * xlo + p.bx, s1 = p.sfx * xhi + p.bx;
        const double t0 = p.sfy * ylo + p.by, t1 = p.sfy * yhi + p.by;
        const double ds = fabs(p.sfx) * dxn + 1e-9 * (fabs(p.bx) + 1.0);
        const double dt = fabs(p.sfy) * dyn + 1e-9 * (fabs(p.by) + 1.0);
        const bool out_s = (fmax(s0, s1) + ds < 0.0) || (fmin(s0, s1) - ds > 1.0);
        const bool out_t = (fmax(t0, t1) + dt < 0.0) || (fmin(t0, t1) - dt > 1.0);
        const bool out_w = (xhi + dxn < -1.0) || (xlo - dxn > 1.0) || (yhi + dyn < -1.0) || (ylo - dyn > 1.0);
        if (out_s || out_t || out_w) keep = 0;
    }
    const unsigned word = __ballot_sync(0xffffffffu, live && keep);
    if ((threadIdx.x & 31) == 0 && live) bits[t >> 5] = word;
    // Footprint tiles (TILE_W x TILE_H texels): every texel a flagged triangle can own lies in its
    // raster bbox (the same tri_bbox the rasteriser used), so the marked tiles cover every texel
    // this stroke can touch; the stream kernel never reads the others.
    if (tile_bits && live && keep) mark_tiles(tri_xy + 6 * t, width, height, row0, rows, tile_bits);
}

// flag lookup in the classification bitmap (global or shared memory); NULL bitmap = keep all
ML_DEV bool tri_flag(const uint32_t* bits, int t) { return bits ? ((bits[t >> 5] >> (t & 31)) & 1u) != 0 : true; }

// Per-triangle record of the TEA evaluation (144 bytes = 9 x 16, written once per camera by
// tea_prepare_kernel): CCW-normalised uv vertices (KN:32-41) and the clip coordinates widened to
// float64 in CCW vertex order (KN:40).  The evaluation fetches it with nine independent 128-bit
// loads instead of 18 scalar gathers behind the winding test.
struct __align__(16) TeaRec {
    double x0, y0, x1, y1, x2, y2;
    double c[12];                     // c0.xyzw, c1.xyzw, c2.xyzw (CCW order)
};
static_assert(sizeof(TeaRec) == 144, "TeaRec is nine 16-byte words");

// Conservative NDC bounds of a triangle for the per-stroke classification, float32 rounded OUTWARD
// (16 bytes per triangle instead of the 96-byte clip record): [x] = xlo - dxn, [y] = xhi + dxn,
// [z] = ylo - dyn, [w] = yhi + dyn with the margins of tea_classify_kernel; an empty interval
// (+inf, -inf) = no fragment can pass (all w <= 0), (-inf, +inf) = always evaluate (mixed signs of w).
template <typename T>
ML_DEV float4 tea_bounds(const T* __restrict__ c) {
    const float inf = __int_as_float(0x7f800000);
    double x[3], y[3], w[3];
#pragma unroll
    for (int v = 0; v < 3; ++v) { x[v] = (double)c[4 * v]; y[v] = (double)c[4 * v + 1]; w[v] = (double)c[4 * v + 3]; }
    const int npos = (w[0] > 0.0) + (w[1] > 0.0) + (w[2] > 0.0);
    const int nnonpos = (w[0] <= 0.0) + (w[1] <= 0.0) + (w[2] <= 0.0);
    if (nnonpos == 3) return make_float4(inf, -inf, inf, -inf);
    if (npos != 3) return make_float4(-inf, inf, -inf, inf);
    const double wmin = fmin(fmin(w[0], w[1]), w[2]);
    const double ax = fmax(fmax(fabs(x[0]), fabs(x[1])), fabs(x[2])) / wmin;
    const double ay = fmax(fmax(fabs(y[0]), fabs(y[1])), fabs(y[2])) / wmin;
    const double xn0 = x[0] / w[0], xn1 = x[1] / w[1], xn2 = x[2] / w[2];
    const double yn0 = y[0] / w[0], yn1 = y[1] / w[1], yn2 = y[2] / w[2];
    const double dxn = 1e-9 * (1.0 + ax), dyn = 1e-9 * (1.0 + ay);
    return make_float4(__double2float_rd(fmin(fmin(xn0, xn1), xn2) - dxn), __double2float_ru(fmax(fmax(xn0, xn1), xn2) + dxn),
                       __double2float_rd(fmin(fmin(yn0, yn1), yn2) - dyn), __double2float_ru(fmax(fmax(yn0, yn1), yn2) + dyn));
}

template <typename T>
__global__ void __launch_bounds__(BLOCK)
tea_prepare_kernel(const T* __restrict__ tri_xy, const T* __restrict__ tri_clip, long long ntri,
                   TeaRec* __restrict__ recs, float4* __restrict__ bounds) {
    const long long t = (long long)blockIdx.x * BLOCK + threadIdx.x;
    if (t >= ntri) return;
    const T* c = tri_clip + 12 * t;
    bounds[t] = tea_bounds(c);
    TriSetup s;
    if (!tri_load_ccw(tri_xy + 6 * t, s)) return;     // degenerate / non-finite: owns no texel, record never read
    TeaRec& r = recs[t];
    r.x0 = s.x0; r.y0 = s.y0; r.x1 = s.x1; r.y1 = s.y1; r.x2 = s.x2; r.y2 = s.y2;
    const int i1 = s.swapped ? 8 : 4, i2 = s.swapped ? 4 : 8;
#pragma unroll
    for (int k = 0; k < 4; ++k) { r.c[k] = (double)c[k]; r.c[4 + k] = (double)c[i1 + k]; r.c[8 + k] = (double)c[i2 + k]; }
}

// Classification from the prepared bounds.  Same decision rule as tea_classify_kernel with the
// triangle side of the margins folded into the stored bounds; the per-stroke side (rounding of
// s = sfx*xn + bx, at most 2u relative) is covered by ds >= 1e-9 * (|bx| + 1 + |sfx|*(1 + |xlo| + |xhi|)).
// Infinite bounds ("always") make every comparison below false, i.e. keep.
template <typename T>
__global__ void __launch_bounds__(BLOCK)
tea_classify_bounds_kernel(const float4* __restrict__ bounds, long long ntri, TeaParams p, uint32_t* __restrict__ bits,
                           const T* __restrict__ tri_xy, long long width, long long height, long long row0, long long rows,
                           uint32_t* __restrict__ tile_bits) {
    const long long t = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const bool live = t < ntri;
    bool keep = false;
    if (live) {
        const float4 b = __ldg(bounds + t);
        if (b.x <= b.y) {
            const double xlo = b.x, xhi = b.y, ylo = b.z, yhi = b.w;
            const double s0 = p.sfx * xlo + p.bx, s1 = p.sfx * xhi + p.bx;
            const double t0 = p.sfy * ylo + p.by, t1 = p.sfy * yhi + p.by;
            const double ds = 1e-9 * (fabs(p.bx) + 1.0 + fabs(p.sfx) * (1.0 + fabs(xlo) + fabs(xhi)));
            const double dt = 1e-9 * (fabs(p.by) + 1.0 + fabs(p.sfy) * (1.0 + fabs(ylo) + fabs(yhi)));
            const bool out_s = (fmax(s0, s1) + ds < 0.0) || (fmin(s0, s1) - ds > 1.0);
            const bool out_t = (fmax(t0, t1) + dt < 0.0) || (fmin(t0, t1) - dt > 1.0);
            const bool out_w = (xhi < -1.0) || (xlo > 1.0) || (yhi < -1.0) || (ylo > 1.0);
            keep = !(out_s || out_t || out_w);
        }
    }
    const unsigned word = __ballot_sync(0xffffffffu, keep);
    if ((threadIdx.x & 31) == 0 && live) bits[t >> 5] = word;
    if (tile_bits && keep) mark_tiles(tri_xy + 6 * t, width, height, row0, rows, tile_bits);
}

// Full KN:166-193 evaluation of one covered texel for its owner triangle.  `recs` (may be NULL)
// are the prepared per-triangle records; both branches compute the same bits.
template <typename T>
ML_DEV bool tea_texel_eval_inline(const T* __restrict__ tri_xy, const T* __restrict__ tri_clip,
                                  const TeaRec* __restrict__ recs, int t, int x, int y, const TeaParams& p) {
    if (recs) {
        // record words: 0..2 = uv vertices, 3/5/7 = (x, y) and 4/6/8 = (z, w) of clip vertices 0/1/2;
        // fetched in three rounds in the order the arithmetic consumes them (register pressure)
        const double2* rp = (const double2*)(recs + t);
        const double2 v0 = __ldg(rp), v1 = __ldg(rp + 1), v2 = __ldg(rp + 2);
        const double2 zw0 = __ldg(rp + 4), zw1 = __ldg(rp + 6), zw2 = __ldg(rp + 8);
        const double cx = xadd((double)x, 0.5), cy = xadd((double)y, 0.5);                                    // KN:60, 63
        const double e0 = xsub(xmul(xsub(v2.x, v1.x), xsub(cy, v1.y)), xmul(xsub(v2.y, v1.y), xsub(cx, v1.x)));   // KN:72
        const double e1 = xsub(xmul(xsub(v0.x, v2.x), xsub(cy, v2.y)), xmul(xsub(v0.y, v2.y), xsub(cx, v2.x)));   // KN:73
        const double e2 = xsub(xmul(xsub(v1.x, v0.x), xsub(cy, v0.y)), xmul(xsub(v1.y, v0.y), xsub(cx, v0.x)));   // KN:74
        const double esum = xadd(xadd(e0, e1), e2);                                   // KN:166
        const double l0 = xdiv(e0, esum), l1 = xdiv(e1, esum), l2 = xdiv(e2, esum);   // KN:167-169
        const double wc = xadd(xadd(xmul(l0, zw0.y), xmul(l1, zw1.y)), xmul(l2, zw2.y));  // KN:173
        if (!(wc > 0.0)) return false;                                                // KN:174
        const double2 xy0 = __ldg(rp + 3), xy1 = __ldg(rp + 5), xy2 = __ldg(rp + 7);
        const double xc = xadd(xadd(xmul(l0, xy0.x), xmul(l1, xy1.x)), xmul(l2, xy2.x));  // KN:170
        const double yc = xadd(xadd(xmul(l0, xy0.y), xmul(l1, xy1.y)), xmul(l2, xy2.y));  // KN:171
        const double zc = xadd(xadd(xmul(l0, zw0.x), xmul(l1, zw1.x)), xmul(l2, zw2.x));  // KN:172
        return tea_filters(p, xc, yc, zc, wc);
    }
    TriSetup s;
    tri_load_ccw(tri_xy + 6ll * t, s);
    double e0, e1, e2;
    tri_inside(s, x, y, e0, e1, e2);
    const T* c = tri_clip + 12ll * t;
    const int i1 = s.swapped ? 8 : 4, i2 = s.swapped ? 4 : 8;
    double c0[4], c1[4], c2[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) { c0[k] = (double)c[k]; c1[k] = (double)c[i1 + k]; c2[k] = (double)c[i2 + k]; }
    return tea_fragment(p, e0, e1, e2, c0, c1, c2);
}
// Out-of-line copy for the streaming kernels, whose (rarely taken) inline-evaluation path must not
// bloat the hot loop; the EVAL kernel, which does nothing else, uses the inline version.
template <typename T>
__device__ __noinline__ bool tea_texel_eval(const T* __restrict__ tri_xy, const T* __restrict__ tri_clip,
                                            const TeaRec* __restrict__ recs, int t, int x, int y, const TeaParams& p) {
    return tea_texel_eval_inline(tri_xy, tri_clip, recs, t, x, y, p);
}

// Work list of quads that need the float64 evaluation.  Entry = 3 x u64: (quad index << 4) | keep
// bits, then the four owner ids (so the EVAL kernel does not gather them again).
struct TeaWork {
    unsigned long long* entries;     // NULL: evaluate inline in the stream kernel
    unsigned long long* count;       // device counter (zeroed before the stream kernel)
    unsigned long long cap;
    const TeaRec* recs;              // prepared per-triangle records (may be NULL)
};

// Footprint culling (optional; needs width % 128 == 0).  tile_cur: tiles this stroke can touch
// (marked by tea_classify); tile_prev: tiles the previous stroke on this edited plane could touch.
// The TILE kernel below visits one 128x8 tile per warp: unmarked tiles cost one bitmap word, tiles
// of tile_prev get their edited bytes cleared (this replaces the whole-plane reset of the
// EditedAreaMask), tiles of tile_cur are processed like the stream kernel does.
struct TeaCull {
    const uint32_t* tile_cur;        // NULL: no culling (stream every texel, count fragments)
    const uint32_t* tile_prev;       // may be NULL
    int segs_per_row;
    unsigned long long known_fragments;   // covered texels of the slab (a skipping kernel cannot count them)
    int reset_edited;                // stream form only: the kernel clears the edited plane while it streams
};
ML_DEV bool tile_bit(const uint32_t* bits, int tile) { return (__ldg(bits + (tile >> 5)) >> (tile & 31)) & 1u; }

// Shared per-step body of the stream and tile kernels.  Each lane holds U quads (index qs[u], owner
// ids ids[u]; qs[u] >= nq marks "nothing").  Must be called by all 32 lanes of a warp.
//   1. flag lookups of all 4*U owners are issued together (independent loads, shared by
//      neighbouring texels); `keep` = texels of flagged triangles;
//   2. kept quads are appended to the work list with ONE warp-aggregated atomic per call;
//   3. whatever did not fit (or everything, without a list) is evaluated inline.
template <typename T, int ES, int U, bool COUNT_FRAGS>
ML_DEV void tea_process(const long long (&qs)[U], const uint4 (&ids)[U], long long nq, const uint32_t* flags,
                        const TeaWork& wk, const TeaParams& p, const T* __restrict__ tri_xy,
                        const T* __restrict__ tri_clip, long long width, long long row0, bool small,
                        void* __restrict__ data, uint32_t value, uint8_t* __restrict__ mask,
                        uint8_t* __restrict__ edited, int lane, long long& newly, long long& frags) {
    unsigned keep[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        keep[u] = 0;
        if (qs[u] >= nq) continue;
        const int t4[4] = {(int)ids[u].x, (int)ids[u].y, (int)ids[u].z, (int)ids[u].w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (t4[e] >= 0) { if (COUNT_FRAGS) ++frags; if (tri_flag(flags, t4[e])) keep[u] |= 1u << e; }
    }
    if (wk.entries) {
        unsigned bal[U];
        int total = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) { bal[u] = __ballot_sync(0xffffffffu, keep[u] != 0); total += __popc(bal[u]); }
        if (total == 0) return;
        unsigned long long slot = 0;
        if (lane == 0) slot = atomicAdd(wk.count, (unsigned long long)total);
        slot = __shfl_sync(0xffffffffu, slot, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (keep[u]) {
                const unsigned long long at = slot + __popc(bal[u] & ((1u << lane) - 1u));
                if (at < wk.cap) {
                    unsigned long long* e3 = wk.entries + 3 * at;
                    e3[0] = ((unsigned long long)qs[u] << 4) | keep[u];
                    e3[1] = (unsigned long long)ids[u].x | ((unsigned long long)ids[u].y << 32);
                    e3[2] = (unsigned long long)ids[u].z | ((unsigned long long)ids[u].w << 32);
                    keep[u] = 0;
                }
            }
            slot += __popc(bal[u]);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {          // inline evaluation: no list, or list overflow
        if (!keep[u]) continue;
        const long long q = qs[u];
        const int t4[4] = {(int)ids[u].x, (int)ids[u].y, (int)ids[u].z, (int)ids[u].w};
        unsigned hits = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if (!(keep[u] & (1u << e))) continue;
            int x, y;
            texel_xy((q << 2) + e, width, row0, small, x, y);
            if (tea_texel_eval(tri_xy, tri_clip, wk.recs, t4[e], x, y, p)) hits |= 1u << e;
        }
        // exactly one thread owns these 4 texels in this kernel: the read-modify-write of
        // KN:198-202 inside quad_write is race-free
        if (hits) quad_write<(ES > 0 ? ES : 1)>(data, value, mask, edited, q << 2, hits, newly);
    }
}

// STREAM kernel (no culling).  One thread per 4 consecutive texels: a 128-bit streaming load of the
// owner ids (4 B/texel is the whole algorithmic traffic) and a flag lookup per owner.
// BS = threads per block; SMEM = the classification bitmap (nwords 32-bit words) is first copied
// to dynamic shared memory, so the per-texel flag lookup is an LDS instead of a dependent L2 gather.
template <typename T, int ES, int BS, bool SMEM>
__global__ void __launch_bounds__(BS)
tea_stream_kernel(const T* __restrict__ tri_xy, const T* __restrict__ tri_clip, long long width,
                  long long row0, long long n, const int* __restrict__ tri_id,
                  const uint32_t* __restrict__ gbits, long long nwords, TeaParams p, TeaWork wk,
                  void* __restrict__ data, int esize, uint32_t value,
                  uint8_t* __restrict__ mask, uint8_t* __restrict__ edited,
                  unsigned long long* counters) {
    extern __shared__ uint32_t s_bits[];
    constexpr int BLOCK = BS;            // shadows the file-level constant inside this kernel
    const uint32_t* flags = gbits;
    if (SMEM) {
        for (long long k = threadIdx.x; k < nwords; k += BS) s_bits[k] = gbits[k];
        __syncthreads();
        flags = s_bits;
    }
    long long newly = 0, frags = 0;
    const long long tid = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * BLOCK;
    const bool small = n <= 0xffffffffLL && width <= 0xffffffffLL;
    const int lane = threadIdx.x & 31;
    long long done = 0;
    if (ES > 0) {
        const long long nq = n >> 2;
        constexpr int U = 4;
        // block-uniform trip count so that the warp-collective append is convergent
        for (long long base = (long long)blockIdx.x * BLOCK; base < nq; base += nthreads * U) {
            uint4 ids[U];
            long long qs[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                qs[u] = base + u * nthreads + threadIdx.x;
                if (qs[u] < nq) ids[u] = ld_stream((const uint4*)tri_id + qs[u]);
            }
            tea_process<T, ES, U, true>(qs, ids, nq, flags, wk, p, tri_xy, tri_clip, width, row0, small,
                                        data, value, mask, edited, lane, newly, frags);
        }
        done = nq << 2;
    }
    for (long long i = done + tid; i < n; i += nthreads) {
        const int t = tri_id[i];
        if (t < 0) continue;
        ++frags;
        if (!tri_flag(flags, t)) continue;
        int x, y;
        texel_xy(i, width, row0, small, x, y);
        if (!tea_texel_eval(tri_xy, tri_clip, wk.recs, t, x, y, p)) continue;
        if (edited[i] == 0) ++newly;
        store_value(data, esize, i, value);
        mask[i] = 1;
        edited[i] = 1;
    }
    block_count_add(newly, counters);
    block_count_add(frags, counters + 1);
}

// STREAM kernel, bulk-copy form (default for aligned planes with the classification bitmap and a
// work list).  The owner-id map -- 4 B/texel, the whole algorithmic traffic of the pass -- is fetched
// by one producer lane per block with cp.async.bulk into a TS_STAGES x TS_CHUNK shared-memory ring
// (bulk.cuh) that sits beside the triangle bitmap; TS_CW consumer warps read their quads of a chunk
// with 128-bit LDS and release the stage.  The register form above keeps 64 B per thread in flight
// (one 1024-thread block per SM next to the 125 KB bitmap = 64 KB per SM) and, worse, spends ~100
// instructions per quad in the generic tea_process (ncu r2: 60 % issue-active at 44 % of the DRAM
// peak -- issue bound).  This kernel's hot loop is ~30 instructions per quad:
//   * the bitmap is stored one word late (s_bits[0] = 0), so an uncovered texel (id -1 -> word
//     index -1 + 1 = 0, bit 31) reads "not flagged" without a compare / select;
//   * 32-bit offsets relative to the chunk; nothing but the flag lookups, the edited reset and one
//     ballot per quad row in the loop; quads with flagged texels (the stroke's footprint, a few per
//     cent of the atlas) leave through an out-of-line append to the evaluation work list.
// RESET: the kernel also clears the edited plane (SPEC.md:255 EditedAreaMask reset) -- each thread
// zeroes the 4 edited bytes of a quad before the quad can be appended, so the separate 1 B/texel
// memset pass (and its launch) disappears into this stream.
#ifndef ML_TS_STAGES
#define ML_TS_STAGES 3
#endif
#ifndef ML_TS_CW
#define ML_TS_CW 16
#endif
#ifndef ML_TS_QPT
#define ML_TS_QPT 4
#endif
constexpr int TS_STAGES = ML_TS_STAGES;
constexpr int TS_CW = ML_TS_CW;                        // consumer warps
constexpr int TS_QPT = ML_TS_QPT;                      // quads per consumer thread and chunk
constexpr int TS_CT = 32 * TS_CW;                      // consumer threads
constexpr int TS_CHUNK = 16 * TS_CT * TS_QPT;          // bytes of ids per chunk (32 KB = 8192 texels)
constexpr int TS_THREADS = TS_CT + 32;
typedef BulkRing<TS_STAGES, TS_CHUNK> TeaRing;

// out-of-line: a warp in which some lane holds a quad with flagged texels appends those quads to the
// work list (one warp-aggregated atomic); whatever does not fit is evaluated here
template <typename T, int ES>
__device__ __noinline__ void tea_stream_append(unsigned keep, long long q, uint4 ids, const TeaWork wk, const TeaParams& p,
                                               const T* __restrict__ tri_xy, const T* __restrict__ tri_clip,
                                               long long width, long long row0, bool small, void* __restrict__ data,
                                               uint32_t value, uint8_t* __restrict__ mask, uint8_t* __restrict__ edited,
                                               unsigned long long* counters) {
    const int lane = threadIdx.x & 31;
    const unsigned bal = __ballot_sync(0xffffffffu, keep != 0);
    unsigned long long slot = 0;
    if (lane == 0) slot = atomicAdd(wk.count, (unsigned long long)__popc(bal));
    slot = __shfl_sync(0xffffffffu, slot, 0);
    if (!keep) return;
    const unsigned long long at = slot + __popc(bal & ((1u << lane) - 1u));
    if (at < wk.cap) {
        unsigned long long* e3 = wk.entries + 3 * at;
        e3[0] = ((unsigned long long)q << 4) | keep;
        e3[1] = (unsigned long long)ids.x | ((unsigned long long)ids.y << 32);
        e3[2] = (unsigned long long)ids.z | ((unsigned long long)ids.w << 32);
        return;
    }
    const int t4[4] = {(int)ids.x, (int)ids.y, (int)ids.z, (int)ids.w};
    unsigned hits = 0;
    for (int e = 0; e < 4; ++e) {
        if (!(keep & (1u << e))) continue;
        int x, y;
        texel_xy((q << 2) + e, width, row0, small, x, y);
        if (tea_texel_eval(tri_xy, tri_clip, wk.recs, t4[e], x, y, p)) hits |= 1u << e;
    }
    long long newly = 0;
    if (hits) quad_write<ES>(data, value, mask, edited, q << 2, hits, newly);
    if (newly) atomicAdd(counters, (unsigned long long)newly);
}

template <typename T, int ES, bool SMEM, bool RESET, bool COUNT>
__global__ void __launch_bounds__(TS_THREADS, 1)
tea_stream_bulk_kernel(const T* __restrict__ tri_xy, const T* __restrict__ tri_clip, long long width,
                       long long row0, long long n, const int* __restrict__ tri_id,
                       const uint32_t* __restrict__ gbits, long long nwords, TeaParams p, TeaWork wk,
                       void* __restrict__ data, int esize, uint32_t value,
                       uint8_t* __restrict__ mask, uint8_t* __restrict__ edited,
                       unsigned long long* counters, unsigned long long known_frags) {
    extern __shared__ __align__(128) uint8_t ts_smem[];
    TeaRing& ring = *reinterpret_cast<TeaRing*>(ts_smem);
    uint32_t* s_bits = reinterpret_cast<uint32_t*>(ts_smem + sizeof(TeaRing));      // [0] = 0, [1 + k] = gbits[k]
    const long long nq = n >> 2;
    const long long id_bytes = nq << 4;
    const long long nchunks = (id_bytes + TS_CHUNK - 1) / TS_CHUNK;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) ring.init(TS_CW);
    __syncthreads();
    RingPos<TS_STAGES> pos;
    long long frags = 0;
    const bool small = n <= 0xffffffffLL && width <= 0xffffffffLL;
    if (warp == TS_CW) {
        // producer: the id stream starts while the consumers still copy the bitmap
        if (lane == 0) {
            const uint64_t policy = l2_policy_evict_first();
            for (long long c = blockIdx.x; c < nchunks; c += gridDim.x, pos.next()) {
                const long long base = c * TS_CHUNK;
                const unsigned bytes = (unsigned)(id_bytes - base < TS_CHUNK ? id_bytes - base : TS_CHUNK);
                ring.produce(pos, (const uint8_t*)tri_id + base, bytes, policy);
            }
        }
    } else {
        if (SMEM) {
            if (threadIdx.x == 0) s_bits[0] = 0u;
            for (long long k = threadIdx.x; k < nwords; k += TS_CT) s_bits[1 + k] = gbits[k];
            asm volatile("bar.sync 1, %0;" :: "n"(TS_CT) : "memory");                // consumers only
        }
        for (long long c = blockIdx.x; c < nchunks; c += gridDim.x, pos.next()) {
            const long long base = c * TS_CHUNK;
            const unsigned bytes = (unsigned)(id_bytes - base < TS_CHUNK ? id_bytes - base : TS_CHUNK);
            const uint8_t* b = ring.acquire(pos);
            uint4 ids[TS_QPT];
#pragma unroll
            for (int u = 0; u < TS_QPT; ++u) {
                const unsigned off = (unsigned)(u * TS_CT + threadIdx.x) << 4;
                ids[u] = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
                if (off < bytes) ids[u] = *(const uint4*)(b + off);
            }
            ring.release(pos);
            uint8_t* ed = edited + (base >> 2);                        // the chunk's edited bytes
            const long long q0 = base >> 4;                            // the chunk's first quad
#pragma unroll
            for (int u = 0; u < TS_QPT; ++u) {
                const unsigned qo = (unsigned)(u * TS_CT + threadIdx.x);           // quad offset in the chunk
                const int t0 = (int)ids[u].x, t1 = (int)ids[u].y, t2 = (int)ids[u].z, t3 = (int)ids[u].w;
                unsigned keep;
                if (SMEM) {
                    keep = (__funnelshift_r(s_bits[1 + (t0 >> 5)], 0u, (unsigned)t0) & 1u)
                         | ((__funnelshift_r(s_bits[1 + (t1 >> 5)], 0u, (unsigned)t1) & 1u) << 1)
                         | ((__funnelshift_r(s_bits[1 + (t2 >> 5)], 0u, (unsigned)t2) & 1u) << 2)
                         | ((__funnelshift_r(s_bits[1 + (t3 >> 5)], 0u, (unsigned)t3) & 1u) << 3);
                } else {
                    keep = (t0 >= 0 ? (__ldg(gbits + (t0 >> 5)) >> (t0 & 31)) & 1u : 0u)
                         | ((t1 >= 0 ? (__ldg(gbits + (t1 >> 5)) >> (t1 & 31)) & 1u : 0u) << 1)
                         | ((t2 >= 0 ? (__ldg(gbits + (t2 >> 5)) >> (t2 & 31)) & 1u : 0u) << 2)
                         | ((t3 >= 0 ? (__ldg(gbits + (t3 >> 5)) >> (t3 & 31)) & 1u : 0u) << 3);
                }
                const bool present = (qo << 4) < bytes;
                if (COUNT) {
                    if ((t0 | t1 | t2 | t3) >= 0) frags += 4;
                    else if (present) frags += 4 + ((t0 >> 31) + (t1 >> 31) + (t2 >> 31) + (t3 >> 31));
                }
                if (RESET && present) *(uint32_t*)(ed + (qo << 2)) = 0u;
                if (__any_sync(0xffffffffu, keep != 0))
                    tea_stream_append<T, ES>(keep, q0 + qo, ids[u], wk, p, tri_xy, tri_clip, width, row0, small,
                                             data, value, mask, edited, counters);
            }
        }
        // tail (n % 4 texels) by the first consumer threads of block 0
        if (blockIdx.x == 0) {
            long long newly = 0;
            for (long long i = (nq << 2) + threadIdx.x; i < n; i += TS_CT) {
                if (RESET) edited[i] = 0;
                const int t = tri_id[i];
                if (t < 0) continue;
                if (COUNT) ++frags;
                if (!tri_flag(gbits, t)) continue;
                int x, y;
                texel_xy(i, width, row0, small, x, y);
                if (!tea_texel_eval(tri_xy, tri_clip, wk.recs, t, x, y, p)) continue;
                if (edited[i] == 0) ++newly;
                store_value(data, esize, i, value);
                mask[i] = 1;
                edited[i] = 1;
            }
            if (newly) atomicAdd(counters, (unsigned long long)newly);
        }
    }
    if (COUNT) block_count_add(frags, counters + 1);
    else if (blockIdx.x == 0 && threadIdx.x == 0 && known_frags) atomicAdd(counters + 1, known_frags);
}

// TILE kernel (footprint culling).  One WARP per LISTED 128x8-texel tile: first the tiles of the
// previous stroke that this stroke does not revisit get their edited bytes cleared (this replaces
// the whole-plane reset of the EditedAreaMask), then every tile of this stroke's list
// is cleared if the previous stroke marked it and streams its 8 row segments (8 independent 128-bit
// id loads per lane) through tea_process.  The stroke therefore reads O(footprint) texels, not
// O(atlas), and the listed tiles spread evenly over the grid wherever the footprint lies.
#ifndef ML_TEA_TILE_MINB
#define ML_TEA_TILE_MINB 3
#endif
template <typename T, int ES>
__global__ void __launch_bounds__(BLOCK, ML_TEA_TILE_MINB)
tea_tile_kernel(const T* __restrict__ tri_xy, const T* __restrict__ tri_clip, long long width,
                long long row0, long long rows, const int* __restrict__ tri_id,
                const uint32_t* __restrict__ flags, TeaParams p, TeaWork wk, TeaCull cull,
                void* __restrict__ data, uint32_t value, uint8_t* __restrict__ mask,
                uint8_t* __restrict__ edited, unsigned long long* counters) {
    constexpr int U = 4;                                   // a warp takes HALF a tile (4 of its 8 rows) per step:
    constexpr int HALVES = (1 << TILE_H_SHIFT) / U;        // fewer registers, three blocks per SM
    long long newly = 0, frags = 0;
    const int lane = threadIdx.x & 31;
    const long long n = rows * width, nq = n >> 2;
    const bool small = n <= 0xffffffffLL && width <= 0xffffffffLL;
    const int segs = cull.segs_per_row;
    const long long ntiles = (long long)segs * ((rows + (1 << TILE_H_SHIFT) - 1) >> TILE_H_SHIFT);
    const TileBuf cur((uint32_t*)cull.tile_cur, ntiles), prev((uint32_t*)cull.tile_prev, ntiles);
    const long long ncur = (long long)*cur.count, nprev = cull.tile_prev ? (long long)*prev.count : 0;
    const long long nwarps = (long long)gridDim.x * (BLOCK / 32);
    for (long long jj = (long long)blockIdx.x * (BLOCK / 32) + (threadIdx.x >> 5); jj < (ncur + nprev) * HALVES; jj += nwarps) {
        const long long j = jj / HALVES;
        const int half = (int)(jj - j * HALVES);
        const bool is_cur = j < ncur;
        const int tile = (int)(is_cur ? cur.list[j] : prev.list[j - ncur]);
        const bool in_prev = cull.tile_prev && tile_bit(prev.bits, tile);
        if (!is_cur && tile_bit(cur.bits, tile)) continue;           // handled by its entry in this stroke's list
        const int ty = tile / segs, tx = tile - ty * segs;
        long long qs[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long yy = ((long long)ty << TILE_H_SHIFT) + half * U + u;
            qs[u] = yy < rows ? ((yy * width + ((long long)tx << TILE_W_SHIFT)) >> 2) + lane : nq;
        }
        if (in_prev || !is_cur) {
#pragma unroll
            for (int u = 0; u < U; ++u) if (qs[u] < nq) *(uint32_t*)(edited + (qs[u] << 2)) = 0u;
        }
        if (!is_cur) continue;
        uint4 ids[U];
#pragma unroll
        for (int u = 0; u < U; ++u) if (qs[u] < nq) ids[u] = ld_stream((const uint4*)tri_id + qs[u]);
        tea_process<T, ES, U, false>(qs, ids, nq, flags, wk, p, tri_xy, tri_clip, width, row0, small,
                                     data, value, mask, edited, lane, newly, frags);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) frags = (long long)cull.known_fragments;
    block_count_add(newly, counters);
    block_count_add(frags, counters + 1);
}

// EVAL kernel.  Four adjacent lanes share one work-list quad, one lane per texel, so the float64
// evaluation runs with full, evenly spread parallelism no matter how compact the tool footprint is
// in atlas space.  The 4 hit bits are gathered with a ballot and lane 0 of the group writes.
#ifndef ML_TEA_EVAL_MINB
#define ML_TEA_EVAL_MINB 4
#endif
template <typename T, int ES>
__global__ void __launch_bounds__(BLOCK, ML_TEA_EVAL_MINB)
tea_eval_kernel(const T* __restrict__ tri_xy, const T* __restrict__ tri_clip, const TeaRec* __restrict__ recs,
                long long width, long long row0, long long n, const int* __restrict__ tri_id, TeaParams p, TeaWork wk,
                void* __restrict__ data, uint32_t value, uint8_t* __restrict__ mask,
                uint8_t* __restrict__ edited, unsigned long long* counters) {
    long long newly = 0;
    const unsigned long long have = *wk.count;
    const long long count = (long long)(have < wk.cap ? have : wk.cap);
    const bool small = n <= 0xffffffffLL && width <= 0xffffffffLL;
    const int lane = threadIdx.x & 31, e = lane & 3;
    const long long nthreads = (long long)gridDim.x * BLOCK;
    const long long step = nthreads >> 2;                 // entries between two iterations of a thread
    // Two-deep software pipeline over the work list: while entry i is evaluated, entry i+1 is already
    // in registers (its triangle record is being prefetched into L1) and the loads of entry i+2 are
    // in flight, so neither the list read nor the record gather sits on the dependent-load chain.
    struct Entry { unsigned long long w, idw; };
    auto load_entry = [&](long long ent) {
        Entry r{0ull, 0ull};
        if (ent < count) { r.w = wk.entries[3 * ent]; r.idw = wk.entries[3 * ent + 1 + (e >> 1)]; }
        return r;
    };
    auto owner = [&](const Entry& en) { return (int)((e & 1) ? (en.idw >> 32) : (en.idw & 0xffffffffull)); };
    auto prefetch_rec = [&](const Entry& en) {
        if (recs && (en.w & (1ull << e))) {
            const char* a = (const char*)(recs + owner(en));
            asm volatile("prefetch.global.L1 [%0];" :: "l"(a));
            asm volatile("prefetch.global.L1 [%0];" :: "l"(a + 128));
        }
    };
    long long ent = ((long long)blockIdx.x * BLOCK + threadIdx.x) >> 2;
    Entry cur = load_entry(ent), nxt = load_entry(ent + step);
    prefetch_rec(cur);
    // block-uniform trip count: every lane reaches the ballot
    for (long long base = (long long)blockIdx.x * BLOCK; base < count * 4; base += nthreads, ent += step) {
        const Entry nn = load_entry(ent + 2 * step);
        prefetch_rec(nxt);
        bool hit = false;
        const long long q = (long long)(cur.w >> 4);
        if (cur.w & (1ull << e)) {
            int x, y;
            texel_xy((q << 2) + e, width, row0, small, x, y);
            hit = tea_texel_eval_inline(tri_xy, tri_clip, recs, owner(cur), x, y, p);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, hit);
        const unsigned hits = (bal >> (lane & ~3)) & 0xfu;
        if (e == 0 && hits) quad_write<ES>(data, value, mask, edited, q << 2, hits, newly);
        cur = nxt;
        nxt = nn;
    }
    block_count_add(newly, counters);
}

inline unsigned grid_for(long long n) {
    long long blocks = (n + BLOCK - 1) / BLOCK;
    const long long cap = (long long)ml_sm_count() * 32;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (unsigned)blocks;
}

inline bool tea_register_stream() {                   // ML_TEA_REGISTER_STREAM: the round-1 stream kernel, kept for comparison
    static const bool v = getenv("ML_TEA_REGISTER_STREAM") != nullptr;
    return v;
}

constexpr int TEA_BIG_BLOCK = 1024;                  // block size when the bitmap lives in shared memory
constexpr long long TEA_SMEM_MAX_BYTES = 200 * 1024; // bitmap size limit for the shared-memory path

template <typename T, int ES>
int launch_tea_es(const T* tri_xy, const T* tri_clip, const TeaRec* recs, long long width, long long row0, long long n,
                  const int* tri_id, const uint32_t* bits, long long ntri, const TeaParams& p, TeaWork wk, TeaCull cull,
                  void* data, int esize, uint32_t value, uint8_t* mask, uint8_t* edited,
                  unsigned long long* ctr, cudaStream_t st) {
    const long long nwords = (ntri + 31) / 32;
    const long long items = ES > 0 ? (n + 15) / 16 : n;     // 4 quads (16 texels) per thread iteration
    const bool smem = ES > 0 && bits != nullptr && nwords * 4 <= TEA_SMEM_MAX_BYTES;
    if (ES > 0 && cull.tile_cur) {
        const long long rows = n / width;
        const long long ntiles = (long long)cull.segs_per_row * ((rows + (1 << TILE_H_SHIFT) - 1) >> TILE_H_SHIFT);
        long long blocks = (2 * ntiles + BLOCK / 32 - 1) / (BLOCK / 32);  // the lists are never longer than this (half tiles)
        const long long cap = (long long)ml_sm_count() * 12;
        if (blocks > cap) blocks = cap;
        if (blocks < 1) blocks = 1;
        tea_tile_kernel<T, (ES > 0 ? ES : 1)><<<(unsigned)blocks, BLOCK, 0, st>>>(tri_xy, tri_clip, width, row0, rows,
            tri_id, bits, p, wk, cull, data, value, mask, edited, ctr);
    } else if (ES > 0 && !tea_register_stream() && n >= TS_CHUNK && bits != nullptr && wk.entries != nullptr) {
        // bulk-copy ring form: one block per SM; the bitmap sits in shared memory beside the ring when it fits
        const bool sm_bits = (size_t)(nwords + 1) * 4 + sizeof(TeaRing) + 128 <= (size_t)227 * 1024;
        const size_t shmem = sizeof(TeaRing) + (sm_bits ? (size_t)(nwords + 1) * 4 : 0);
        const long long nchunks = ((n >> 2) * 16 + TS_CHUNK - 1) / TS_CHUNK;
        long long blocks = ml_sm_count();
        if (blocks > nchunks) blocks = nchunks;
        constexpr int E = ES > 0 ? ES : 1;
        const bool count = cull.known_fragments == 0;      // the caller knows the slab's covered-texel count: nothing to recount
#define ML_LAUNCH_TSB(SM, RS, CN) do { \
            auto kern = tea_stream_bulk_kernel<T, E, SM, RS, CN>; \
            ML_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem)); \
            kern<<<(unsigned)blocks, TS_THREADS, shmem, st>>>(tri_xy, tri_clip, width, row0, n, tri_id, bits, nwords, p, wk, \
                data, esize, value, mask, edited, ctr, cull.known_fragments); } while (0)
#define ML_LAUNCH_TSB2(SM, RS) do { if (count) ML_LAUNCH_TSB(SM, RS, true); else ML_LAUNCH_TSB(SM, RS, false); } while (0)
        if (sm_bits) { if (cull.reset_edited) ML_LAUNCH_TSB2(true, true); else ML_LAUNCH_TSB2(true, false); }
        else { if (cull.reset_edited) ML_LAUNCH_TSB2(false, true); else ML_LAUNCH_TSB2(false, false); }
#undef ML_LAUNCH_TSB2
#undef ML_LAUNCH_TSB
    } else if (smem) {
        if (cull.reset_edited) ML_CUDA(cudaMemsetAsync(edited, 0, (size_t)n, st));
        // one 1024-thread block per SM (the bitmap takes most of its shared memory)
        auto kern = tea_stream_kernel<T, ES, TEA_BIG_BLOCK, true>;
        ML_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(nwords * 4)));
        long long blocks = (items + TEA_BIG_BLOCK - 1) / TEA_BIG_BLOCK;
        const long long cap = (long long)ml_sm_count() * (nwords * 4 <= 100 * 1024 ? 2 : 1);
        if (blocks > cap) blocks = cap;
        if (blocks < 1) blocks = 1;
        kern<<<(unsigned)blocks, TEA_BIG_BLOCK, (size_t)(nwords * 4), st>>>(tri_xy, tri_clip, width, row0, n, tri_id,
            bits, nwords, p, wk, data, esize, value, mask, edited, ctr);
    } else {
        if (cull.reset_edited) ML_CUDA(cudaMemsetAsync(edited, 0, (size_t)n, st));
        long long blocks = (items + BLOCK - 1) / BLOCK;
        const long long cap = (long long)ml_sm_count() * 16;
        if (blocks > cap) blocks = cap;
        if (blocks < 1) blocks = 1;
        tea_stream_kernel<T, ES, BLOCK, false><<<(unsigned)blocks, BLOCK, 0, st>>>(tri_xy, tri_clip, width, row0, n,
            tri_id, bits, nwords, p, wk, data, esize, value, mask, edited, ctr);
    }
    if (ES > 0 && wk.entries)
        tea_eval_kernel<T, (ES > 0 ? ES : 1)><<<(unsigned)(ml_sm_count() * 8), BLOCK, 0, st>>>(tri_xy, tri_clip, recs, width,
            row0, n, tri_id, p, wk, data, value, mask, edited, ctr);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

template <typename T>
int launch_tea_texels(const T* tri_xy, const T* tri_clip, const TeaRec* recs, long long width, long long row0, long long n,
                      const int* tri_id, const uint32_t* bits, long long ntri, const TeaParams& p, void* worklist,
                      size_t worklist_bytes, TeaCull cull, void* data, int esize, uint32_t value, uint8_t* mask,
                      uint8_t* edited, unsigned long long* ctr, cudaStream_t st) {
    const bool vec = ((((uintptr_t)tri_id) | ((uintptr_t)data) | ((uintptr_t)mask) | ((uintptr_t)edited)) & 15) == 0;
    TeaWork wk{nullptr, nullptr, 0, recs};
    if (vec && worklist && worklist_bytes >= 64 && (((uintptr_t)worklist) & 7) == 0) {
        wk.count = (unsigned long long*)worklist;
        wk.entries = wk.count + 2;
        wk.cap = (worklist_bytes - 16) / 24;
        ML_CUDA(cudaMemsetAsync(wk.count, 0, 8, st));
    }
    if (!vec || (width & ((1 << TILE_W_SHIFT) - 1)) != 0 || bits == nullptr) {
        if (cull.tile_cur) return ml_fail(ML_ERR_ARG, "footprint culling needs width % 128 == 0, aligned planes and triangle flags");
    }
    cull.segs_per_row = (int)(width >> TILE_W_SHIFT);
    if (!vec) return launch_tea_es<T, 0>(tri_xy, tri_clip, recs, width, row0, n, tri_id, bits, ntri, p, wk, cull, data, esize, value, mask, edited, ctr, st);
    if (esize == 1) return launch_tea_es<T, 1>(tri_xy, tri_clip, recs, width, row0, n, tri_id, bits, ntri, p, wk, cull, data, esize, value, mask, edited, ctr, st);
    if (esize == 2) return launch_tea_es<T, 2>(tri_xy, tri_clip, recs, width, row0, n, tri_id, bits, ntri, p, wk, cull, data, esize, value, mask, edited, ctr, st);
    return launch_tea_es<T, 4>(tri_xy, tri_clip, recs, width, row0, n, tri_id, bits, ntri, p, wk, cull, data, esize, value, mask, edited, ctr, st);
}

}  // namespace

extern "C" {

size_t ml_surface_workspace_bytes(int64_t ntri) {          // records | slab count | slab list
    return (size_t)(ntri > 0 ? ntri : 0) * (sizeof(TriRec) + sizeof(int)) + 64;
}

int ml_surface_resolve(const void* tri_xy, const void* tri_pos, const void* tri_nrm, int tri_dtype,
                       int64_t ntri, int64_t width, int64_t row0, int64_t rows,
                       const int32_t* tri_id, float* pos, float* nrm, float* area,
                       uint64_t* covered, void* workspace, size_t workspace_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const long long n = (long long)rows * width;
    if (n <= 0) return ML_OK;
    if (tri_dtype != ML_F32 && tri_dtype != ML_F64) return ml_fail(ML_ERR_ARG, "tri_dtype must be ML_F32 or ML_F64");
    if (workspace == nullptr || workspace_bytes < ml_surface_workspace_bytes(ntri) || (((uintptr_t)workspace) & 15))
        return ml_fail(ML_ERR_ARG, "surface resolve needs a 16-byte aligned workspace of ml_surface_workspace_bytes(ntri)");
    unsigned long long* ctr = (unsigned long long*)covered;
    TriRec* recs = (TriRec*)workspace;
    const bool small = n <= 0xffffffffLL && width <= 0xffffffffLL;
    const unsigned pgrid = (unsigned)((ntri + BLOCK - 1) / BLOCK);
    if (ntri > 0) {
        const int* slab_list = nullptr;
        const unsigned long long* slab_count = nullptr;
        // the caller's slab geometry is (row0, rows) only; a slab is recognised by the list paying off: rows of the
        // slab against the rows the triangles span is unknown here, so the list is built whenever the mesh is large
        // (0.1 ms per 10 M triangles) and the records of the listed triangles alone are written
        if (ntri >= 4096) {
            unsigned long long* cnt = (unsigned long long*)((char*)workspace + (size_t)ntri * sizeof(TriRec));
            int* list = (int*)(cnt + 2);
            ML_CUDA(cudaMemsetAsync(cnt, 0, 16, st));
            const int rc = ml_slab_triangle_list(tri_xy, tri_dtype, ntri, row0, rows, list, cnt, st);
            if (rc != ML_OK) return rc;
            slab_list = list; slab_count = cnt;
        }
        if (tri_dtype == ML_F32)
            tri_prepare_kernel<float><<<pgrid, BLOCK, 0, st>>>((const float*)tri_xy, (const float*)tri_pos, (const float*)tri_nrm, ntri, recs, slab_list, slab_count);
        else
            tri_prepare_kernel<double><<<pgrid, BLOCK, 0, st>>>((const double*)tri_xy, (const double*)tri_pos, (const double*)tri_nrm, ntri, recs, slab_list, slab_count);
    }
    if (small) resolve_kernel<true><<<grid_for(n), BLOCK, 0, st>>>(recs, width, row0, n, tri_id, pos, nrm, area, ctr);
    else resolve_kernel<false><<<grid_for(n), BLOCK, 0, st>>>(recs, width, row0, n, tri_id, pos, nrm, area, ctr);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int ml_tea_tile_words(int64_t width, int64_t rows) {
    if (width <= 0 || rows <= 0 || (width & ((1 << TILE_W_SHIFT) - 1)) != 0) return 0;
    const long long tiles = (width >> TILE_W_SHIFT) * ((rows + (1 << TILE_H_SHIFT) - 1) >> TILE_H_SHIFT);
    return (int)(tile_bitmap_words(tiles) + 2 + tiles);             // bitmap | count | list (TileBuf)
}

int ml_tea_classify(const void* tri_clip, int tri_dtype, int64_t ntri, const ml_tea_params* tp,
                    uint32_t* flags, const void* tri_xy, int64_t width, int64_t height, int64_t row0,
                    int64_t rows, uint32_t* tile_bits, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (ntri <= 0) return ML_OK;
    TeaParams p = ml_make_tea_params(tp);
    if (tile_bits) {
        const int words = ml_tea_tile_words(width, rows);
        if (words == 0 || tri_xy == nullptr) return ml_fail(ML_ERR_ARG, "tile marking needs tri_xy and width % 128 == 0");
        const long long tiles = (width >> TILE_W_SHIFT) * ((rows + (1 << TILE_H_SHIFT) - 1) >> TILE_H_SHIFT);
        ML_CUDA(cudaMemsetAsync(tile_bits, 0, (size_t)(tile_bitmap_words(tiles) + 2) * 4, st));   // bitmap + list count
    }
    const unsigned grid = (unsigned)((ntri + BLOCK - 1) / BLOCK);
    if (tri_dtype == ML_F32) tea_classify_kernel<float><<<grid, BLOCK, 0, st>>>((const float*)tri_clip, ntri, p, flags, (const float*)tri_xy, width, height, row0, rows, tile_bits);
    else if (tri_dtype == ML_F64) tea_classify_kernel<double><<<grid, BLOCK, 0, st>>>((const double*)tri_clip, ntri, p, flags, (const double*)tri_xy, width, height, row0, rows, tile_bits);
    else return ml_fail(ML_ERR_ARG, "tri_dtype must be ML_F32 or ML_F64");
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

// record buffer = [TeaRec x ntri][float4 bounds x ntri]
size_t ml_tea_rec_bytes(int64_t ntri) { return (size_t)(ntri > 0 ? ntri : 0) * (sizeof(TeaRec) + sizeof(float4)) + 16; }
static inline float4* tea_bounds_of(const void* recs, int64_t ntri) { return (float4*)((char*)recs + (size_t)ntri * sizeof(TeaRec)); }

int ml_tea_prepare(const void* tri_xy, const void* tri_clip, int tri_dtype, int64_t ntri, void* recs,
                   size_t rec_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (ntri <= 0) return ML_OK;
    if (recs == nullptr || rec_bytes < ml_tea_rec_bytes(ntri) || (((uintptr_t)recs) & 15))
        return ml_fail(ML_ERR_ARG, "ml_tea_prepare needs ml_tea_rec_bytes(ntri) bytes, 16-byte aligned");
    const unsigned grid = (unsigned)((ntri + BLOCK - 1) / BLOCK);
    if (tri_dtype == ML_F32) tea_prepare_kernel<float><<<grid, BLOCK, 0, st>>>((const float*)tri_xy, (const float*)tri_clip, ntri, (TeaRec*)recs, tea_bounds_of(recs, ntri));
    else if (tri_dtype == ML_F64) tea_prepare_kernel<double><<<grid, BLOCK, 0, st>>>((const double*)tri_xy, (const double*)tri_clip, ntri, (TeaRec*)recs, tea_bounds_of(recs, ntri));
    else return ml_fail(ML_ERR_ARG, "tri_dtype must be ML_F32 or ML_F64");
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int ml_tea_classify_recs(const void* tea_recs, int tri_dtype, int64_t ntri, const ml_tea_params* tp,
                         uint32_t* flags, const void* tri_xy, int64_t width, int64_t height, int64_t row0,
                         int64_t rows, uint32_t* tile_bits, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (ntri <= 0) return ML_OK;
    if (tea_recs == nullptr) return ml_fail(ML_ERR_ARG, "ml_tea_classify_recs needs the records of ml_tea_prepare");
    TeaParams p = ml_make_tea_params(tp);
    if (tile_bits) {
        const int words = ml_tea_tile_words(width, rows);
        if (words == 0 || tri_xy == nullptr) return ml_fail(ML_ERR_ARG, "tile marking needs tri_xy and width % 128 == 0");
        const long long tiles = (width >> TILE_W_SHIFT) * ((rows + (1 << TILE_H_SHIFT) - 1) >> TILE_H_SHIFT);
        ML_CUDA(cudaMemsetAsync(tile_bits, 0, (size_t)(tile_bitmap_words(tiles) + 2) * 4, st));   // bitmap + list count
    }
    const unsigned grid = (unsigned)((ntri + BLOCK - 1) / BLOCK);
    const float4* bounds = tea_bounds_of(tea_recs, ntri);
    if (tri_dtype == ML_F32) tea_classify_bounds_kernel<float><<<grid, BLOCK, 0, st>>>(bounds, ntri, p, flags, (const float*)tri_xy, width, height, row0, rows, tile_bits);
    else if (tri_dtype == ML_F64) tea_classify_bounds_kernel<double><<<grid, BLOCK, 0, st>>>(bounds, ntri, p, flags, (const double*)tri_xy, width, height, row0, rows, tile_bits);
    else return ml_fail(ML_ERR_ARG, "tri_dtype must be ML_F32 or ML_F64");
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int ml_tea_texels(const void* tri_xy, const void* tri_clip, const void* tea_recs, int tri_dtype, int64_t ntri,
                  int64_t width, int64_t row0, int64_t rows, const int32_t* tri_id,
                  const uint32_t* tri_flags, const ml_tea_params* tp, void* worklist,
                  size_t worklist_bytes, const uint32_t* tile_cur, const uint32_t* tile_prev,
                  int64_t known_fragments, void* data, int esize,
                  uint32_t value_bits, uint8_t* mask, uint8_t* edited, uint64_t* counters, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (esize != 1 && esize != 2 && esize != 4) return ml_fail(ML_ERR_ARG, "esize must be 1, 2 or 4");
    const long long n = (long long)rows * width;
    if (n <= 0) return ML_OK;
    TeaParams p = ml_make_tea_params(tp);
    unsigned long long* ctr = (unsigned long long*)counters;
    TeaCull cull{tile_cur, tile_cur ? tile_prev : nullptr, 0, (unsigned long long)(known_fragments > 0 ? known_fragments : 0), 0};
    if (tri_dtype == ML_F32)
        return launch_tea_texels((const float*)tri_xy, (const float*)tri_clip, (const TeaRec*)tea_recs, width, row0, n, tri_id, tri_flags, ntri, p,
                                 worklist, worklist_bytes, cull, data, esize, value_bits, mask, edited, ctr, st);
    if (tri_dtype == ML_F64)
        return launch_tea_texels((const double*)tri_xy, (const double*)tri_clip, (const TeaRec*)tea_recs, width, row0, n, tri_id, tri_flags, ntri, p,
                                 worklist, worklist_bytes, cull, data, esize, value_bits, mask, edited, ctr, st);
    return ml_fail(ML_ERR_ARG, "tri_dtype must be ML_F32 or ML_F64");
}

int ml_tea_stream(const void* tri_xy, const void* tri_clip, const void* tea_recs, int tri_dtype, int64_t ntri,
                  int64_t width, int64_t row0, int64_t rows, const int32_t* tri_id,
                  const uint32_t* tri_flags, const ml_tea_params* tp, void* worklist, size_t worklist_bytes,
                  int reset_edited, int64_t known_fragments, void* data, int esize, uint32_t value_bits, uint8_t* mask, uint8_t* edited,
                  uint64_t* counters, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (esize != 1 && esize != 2 && esize != 4) return ml_fail(ML_ERR_ARG, "esize must be 1, 2 or 4");
    const long long n = (long long)rows * width;
    if (n <= 0) return ML_OK;
    TeaParams p = ml_make_tea_params(tp);
    unsigned long long* ctr = (unsigned long long*)counters;
    TeaCull cull{nullptr, nullptr, 0, (unsigned long long)(known_fragments > 0 ? known_fragments : 0), reset_edited ? 1 : 0};
    if (tri_dtype == ML_F32)
        return launch_tea_texels((const float*)tri_xy, (const float*)tri_clip, (const TeaRec*)tea_recs, width, row0, n, tri_id, tri_flags, ntri, p,
                                 worklist, worklist_bytes, cull, data, esize, value_bits, mask, edited, ctr, st);
    if (tri_dtype == ML_F64)
        return launch_tea_texels((const double*)tri_xy, (const double*)tri_clip, (const TeaRec*)tea_recs, width, row0, n, tri_id, tri_flags, ntri, p,
                                 worklist, worklist_bytes, cull, data, esize, value_bits, mask, edited, ctr, st);
    return ml_fail(ML_ERR_ARG, "tri_dtype must be ML_F32 or ML_F64");
}

int ml_stroke(const ml_stroke_ctx* c, int cur, const ml_tea_params* tp, void* data, int esize,
              uint32_t value_bits, uint8_t* mask, int64_t padding_radius, uint64_t* counters, void* stream) {
    if (c == nullptr || (cur != 0 && cur != 1)) return ml_fail(ML_ERR_ARG, "ml_stroke: bad context / tile buffer index");
    if (c->tiles[0] == nullptr || c->tiles[1] == nullptr || c->tea_recs == nullptr || c->tri_flags == nullptr)
        return ml_fail(ML_ERR_ARG, "ml_stroke needs the prepared records, the triangle flags and both tile buffers");
    ML_CUDA(cudaMemsetAsync(counters, 0, 3 * sizeof(uint64_t), (cudaStream_t)stream));
    int rc = ml_tea_classify_recs(c->tea_recs, c->tri_dtype, c->ntri, tp, c->tri_flags, c->tri_xy, c->width, c->height,
                                  c->row0, c->rows, c->tiles[cur], stream);
    if (rc != ML_OK) return rc;
    rc = ml_tea_texels(c->tri_xy, c->tri_clip, c->tea_recs, c->tri_dtype, c->ntri, c->width, c->row0, c->rows, c->tri_id,
                       c->tri_flags, tp, c->worklist, c->worklist_bytes, c->tiles[cur], c->tiles[cur ^ 1],
                       c->known_fragments, data, esize, value_bits, mask, c->edited, counters, stream);
    if (rc != ML_OK || padding_radius <= 0 || c->outline == nullptr) return rc;
    return ml_apply_padding_tiles(c->outline, c->edited, c->width, c->rows, padding_radius, c->tiles[cur], data, esize,
                                  value_bits, mask, counters + 2, stream);
}

int ml_stroke_sequence(const ml_stroke_ctx* c, int first_cur, int64_t n, const ml_tea_params* tp, void* data, int esize,
                       const uint32_t* value_bits, uint8_t* mask, int64_t padding_radius, uint64_t* counters,
                       void* stream) {
    if (n < 0 || tp == nullptr || value_bits == nullptr) return ml_fail(ML_ERR_ARG, "ml_stroke_sequence: bad arguments");
    for (int64_t k = 0; k < n; ++k) {
        const int rc = ml_stroke(c, (first_cur + (int)(k & 1)) & 1, tp + k, data, esize, value_bits[k], mask, padding_radius,
                                 counters + 3 * k, stream);
        if (rc != ML_OK) return rc;
    }
    return ML_OK;
}

}  // extern "C"
