// Shared device helpers for libmeshlayers_b200 (sm_100a only).
//
// Arithmetic contract (reference: pkg/src/meshlayers/_kernels_numpy.py:1-25, cited KN:line):
// every decision is taken in IEEE float64 with the reference's exact association order and NO
// fused multiply-add.  The helpers below use the round-to-nearest intrinsics, which ptxas never
// contracts; the library is additionally compiled with -fmad=false.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#define ML_DEV __device__ __forceinline__

ML_DEV double xadd(double a, double b) { return __dadd_rn(a, b); }
ML_DEV double xsub(double a, double b) { return __dsub_rn(a, b); }
ML_DEV double xmul(double a, double b) { return __dmul_rn(a, b); }
ML_DEV double xdiv(double a, double b) { return __ddiv_rn(a, b); }

// ---------------------------------------------------------------------------------------------
// streaming memory access: 128-bit, read-only path, no L1 allocation (each byte is touched once)
ML_DEV uint4 ld_stream(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
// same without .nc: legal when the kernel's output may alias this input (in-place layer ops)
ML_DEV uint4 ld_stream_rw(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
    return r;
}
ML_DEV float4 ld_stream(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
ML_DEV uint32_t ld_stream(const uint32_t* p) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
ML_DEV uint32_t ld_volatile_u32(const uint32_t* p) {
    uint32_t r;
    asm volatile("ld.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
    return r;
}
// streaming load of a 4-element group of 1-, 2- or 4-byte elements (4 / 8 / 16 bytes)
template <typename Q>
ML_DEV Q ld_quad(const Q* p) {
    Q r;
    if (sizeof(Q) == 16) { uint4 v = ld_stream((const uint4*)p); memcpy(&r, &v, 16); }
    else if (sizeof(Q) == 8) {
        uint2 v;
        asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
        memcpy(&r, &v, 8);
    } else { uint32_t v = ld_stream((const uint32_t*)p); memcpy(&r, &v, 4); }
    return r;
}
ML_DEV void st_stream(uint4* p, uint4 v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
ML_DEV void st_stream(uint32_t* p, uint32_t v) {
    asm volatile("st.global.L1::no_allocate.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------------------------------------
// warp / block reductions
ML_DEV long long warp_sum(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
ML_DEV double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = xadd(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
// Block-wide integer sum followed by ONE atomic per block.  Must be reached by all threads.
ML_DEV void block_count_add(long long v, unsigned long long* counter) {
    __shared__ long long s_part[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    if (lane == 0) s_part[wid] = v;
    __syncthreads();
    if (wid == 0) {
        long long t = lane < nw ? s_part[lane] : 0;
        t = warp_sum(t);
        if (lane == 0 && t != 0) atomicAdd(counter, (unsigned long long)t);
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------------------------
// Byte planes (mask / edited / coverage, bool or uint8): set one byte to exactly 1 through a
// 32-bit atomic on the enclosing word and report whether it was 0 before.  This reproduces
// KN:97-99 / KN:198-202 ("count texels that go 0 -> 1, then store 1") under any interleaving
// of writers that target the same texel.
ML_DEV bool byte_set1_was0(uint8_t* plane, long long i) {
    uint8_t* p = plane + i;
    uint8_t cur = *(volatile uint8_t*)p;
    if (cur == 1) return false;
    uintptr_t a = (uintptr_t)p;
    unsigned* w = (unsigned*)(a & ~(uintptr_t)3);
    const unsigned sh = (unsigned)(a & 3) * 8u;
    if (cur == 0) {
        unsigned old = atomicOr(w, 1u << sh);
        unsigned ob = (old >> sh) & 0xffu;
        if (ob == 0) return true;
        if (ob == 1) return false;
    }
    // the byte held some other non-zero value: force it to exactly 1
    unsigned old = *(volatile unsigned*)w, assumed;
    do {
        assumed = old;
        old = atomicCAS(w, assumed, (assumed & ~(0xffu << sh)) | (1u << sh));
    } while (old != assumed);
    return false;
}

// store `esize` (1, 2 or 4) bytes of `bits` at element i of a data plane
ML_DEV void store_value(void* data, int esize, long long i, uint32_t bits) {
    if (esize == 1) ((uint8_t*)data)[i] = (uint8_t)bits;
    else if (esize == 2) ((uint16_t*)data)[i] = (uint16_t)bits;
    else ((uint32_t*)data)[i] = bits;
}

// ---------------------------------------------------------------------------------------------
// Quad write: the KN:198-202 write rule for 4 horizontally adjacent texels owned by ONE thread
// (texel index i is a multiple of 4, planes are 4-byte aligned).  `hits` has bit e set when texel
// i+e is hit.  Byte planes are updated with one 32-bit read-modify-write instead of four byte
// stores (partial-sector byte stores are what makes hit-heavy strokes slow); returns through cnt
// the number of hit texels whose edited flag was 0.
ML_DEV uint32_t spread4(unsigned hits) {            // 4 bits -> 4 byte lanes of 0xff
    return ((hits * 0x00204081u) & 0x01010101u) * 0xffu;
}
ML_DEV uint32_t zero_bytes_msb(uint32_t w) {        // bit 7 of each byte lane set iff that byte == 0
    return ~((((w & 0x7f7f7f7fu) + 0x7f7f7f7fu) | w)) & 0x80808080u;
}
ML_DEV unsigned nz_bits4(uint32_t w) {             // 4-bit mask of the non-zero byte lanes of a word
    const uint32_t nz = (~zero_bytes_msb(w) & 0x80808080u) >> 7;          // bits 0, 8, 16, 24
    return ((nz * 0x00204081u) >> 21) & 0xfu;
}
// The write is split in two so that a thread holding several hit quads can issue ALL its old-word
// loads before the first store (independent loads overlap; a load behind a store to a may-alias
// plane would serialise a DRAM round trip per plane per quad):
//   quad_load   : edited word (always, for the 0 -> 1 count); mask and 1-byte data words only when
//                 the quad is partially hit (a fully hit quad overwrites them).
//   quad_commit : merge + store, skipping stores that would not change the word.
template <int ES>
ML_DEV void quad_load(const void* data, const uint8_t* mask, const uint8_t* edited, long long i,
                      unsigned hits, uint32_t& ew, uint32_t& mw, uint32_t& dw) {
    ew = 0u; mw = 0u; dw = 0u;
    if (!hits) return;
    ew = *(const uint32_t*)(edited + i);
    if (hits != 0xfu) {
        mw = *(const uint32_t*)(mask + i);
        if (ES == 1) dw = *(const uint32_t*)((const uint8_t*)data + i);
    }
}
template <int ES>
ML_DEV void quad_commit(void* data, uint32_t value, uint8_t* mask, uint8_t* edited, long long i,
                        unsigned hits, uint32_t ew, uint32_t mw, uint32_t dw, long long& cnt) {
    if (!hits) return;
    const uint32_t hm = spread4(hits);
    cnt += __popc(zero_bytes_msb(ew) & hm);
    const uint32_t en = (ew & ~hm) | (0x01010101u & hm);
    if (en != ew) *(uint32_t*)(edited + i) = en;
    uint32_t* pm = (uint32_t*)(mask + i);
    if (hits == 0xfu) *pm = 0x01010101u;
    else { const uint32_t mn = (mw & ~hm) | (0x01010101u & hm); if (mn != mw) *pm = mn; }
    if (ES == 1) {
        uint32_t* pd = (uint32_t*)((uint8_t*)data + i);
        const uint32_t vr = (value & 0xffu) * 0x01010101u;
        if (hits == 0xfu) *pd = vr;
        else { const uint32_t dn = (dw & ~hm) | (vr & hm); if (dn != dw) *pd = dn; }
    } else if (ES == 2) {
        uint16_t* pd = (uint16_t*)data + i;
        if (hits == 0xfu) { const uint32_t vr = (value & 0xffffu) * 0x00010001u; *(uint2*)pd = make_uint2(vr, vr); }
        else {
#pragma unroll
            for (int e = 0; e < 4; ++e) if (hits & (1u << e)) pd[e] = (uint16_t)value;
        }
    } else {
        uint32_t* pd = (uint32_t*)data + i;
        if (hits == 0xfu) *(uint4*)pd = make_uint4(value, value, value, value);
        else {
#pragma unroll
            for (int e = 0; e < 4; ++e) if (hits & (1u << e)) pd[e] = value;
        }
    }
}
template <int ES>
ML_DEV void quad_write(void* data, uint32_t value, uint8_t* mask, uint8_t* edited, long long i,
                       unsigned hits, long long& cnt) {
    uint32_t ew, mw, dw;
    quad_load<ES>(data, mask, edited, i, hits, ew, mw, dw);
    quad_commit<ES>(data, value, mask, edited, i, hits, ew, mw, dw, cnt);
}

// 16-texel form of the quad write for threads that own 16 consecutive texels (i0 % 16 == 0, planes
// 16-byte aligned): the byte planes move as ONE 128-bit access per plane and thread instead of four
// 32-bit ones (a quarter of the memory instructions, 512 contiguous bytes per warp access).  hit16
// bit e <-> texel i0 + e.  Same rule as quad_load / quad_commit: edited is always read (0 -> 1
// count), mask / 1-byte data only when the vector is partially hit.
template <int ES>
ML_DEV void vec16_load(const void* data, const uint8_t* mask, const uint8_t* edited, long long i0,
                       unsigned hit16, uint4& ew, uint4& mw, uint4& dw) {
    ew = mw = dw = make_uint4(0u, 0u, 0u, 0u);
    if (!hit16) return;
    ew = *(const uint4*)(edited + i0);
    if (hit16 != 0xffffu) {
        mw = *(const uint4*)(mask + i0);
        if (ES == 1) dw = *(const uint4*)((const uint8_t*)data + i0);
    }
}
ML_DEV uint32_t merge_word(uint32_t old, uint32_t hm, uint32_t rep) { return (old & ~hm) | (rep & hm); }
template <int ES>
ML_DEV void vec16_commit(void* data, uint32_t value, uint8_t* mask, uint8_t* edited, long long i0,
                         unsigned hit16, const uint4& ew, const uint4& mw, const uint4& dw, long long& cnt) {
    if (!hit16) return;
    const uint32_t h0 = spread4(hit16 & 0xfu), h1 = spread4((hit16 >> 4) & 0xfu),
                   h2 = spread4((hit16 >> 8) & 0xfu), h3 = spread4((hit16 >> 12) & 0xfu);
    cnt += __popc(zero_bytes_msb(ew.x) & h0) + __popc(zero_bytes_msb(ew.y) & h1) +
           __popc(zero_bytes_msb(ew.z) & h2) + __popc(zero_bytes_msb(ew.w) & h3);
    const uint32_t one = 0x01010101u;
    const uint4 en = make_uint4(merge_word(ew.x, h0, one), merge_word(ew.y, h1, one), merge_word(ew.z, h2, one), merge_word(ew.w, h3, one));
    if ((en.x ^ ew.x) | (en.y ^ ew.y) | (en.z ^ ew.z) | (en.w ^ ew.w)) *(uint4*)(edited + i0) = en;
    if (hit16 == 0xffffu) *(uint4*)(mask + i0) = make_uint4(one, one, one, one);
    else {
        const uint4 mn = make_uint4(merge_word(mw.x, h0, one), merge_word(mw.y, h1, one), merge_word(mw.z, h2, one), merge_word(mw.w, h3, one));
        if ((mn.x ^ mw.x) | (mn.y ^ mw.y) | (mn.z ^ mw.z) | (mn.w ^ mw.w)) *(uint4*)(mask + i0) = mn;
    }
    if (ES == 1) {
        const uint32_t vr = (value & 0xffu) * 0x01010101u;
        if (hit16 == 0xffffu) *(uint4*)((uint8_t*)data + i0) = make_uint4(vr, vr, vr, vr);
        else {
            const uint4 dn = make_uint4(merge_word(dw.x, h0, vr), merge_word(dw.y, h1, vr), merge_word(dw.z, h2, vr), merge_word(dw.w, h3, vr));
            if ((dn.x ^ dw.x) | (dn.y ^ dw.y) | (dn.z ^ dw.z) | (dn.w ^ dw.w)) *(uint4*)((uint8_t*)data + i0) = dn;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const unsigned hits = (hit16 >> (4 * j)) & 0xfu;
            if (!hits) continue;
            const long long i = i0 + 4 * j;
            if (ES == 2) {
                uint16_t* pd = (uint16_t*)data + i;
                if (hits == 0xfu) { const uint32_t vr = (value & 0xffffu) * 0x00010001u; *(uint2*)pd = make_uint2(vr, vr); }
                else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) if (hits & (1u << e)) pd[e] = (uint16_t)value;
                }
            } else {
                uint32_t* pd = (uint32_t*)data + i;
                if (hits == 0xfu) *(uint4*)pd = make_uint4(value, value, value, value);
                else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) if (hits & (1u << e)) pd[e] = value;
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------------------------
// Triangle setup: KN:32-41 (_ccw), KN:44-47 (tie rule), KN:50-59 (bbox, tightened).
struct TriSetup {
    double x0, y0, x1, y1, x2, y2;   // CCW-normalised vertices, grid units
    double ax, ay, bx, by, cx, cy;   // edge deltas: a = v2-v1, b = v0-v2, c = v1-v0
    int ix0, ix1, iy0, iy1;          // inclusive texel bbox, clipped to the plane / row slab
    bool t0, t1, t2;                 // edge i accepts e == 0
    bool swapped;                    // vertices 1 and 2 were exchanged
};

template <typename T>
ML_DEV bool tri_load_ccw(const T* __restrict__ xy, TriSetup& s) {
    double x0 = (double)xy[0], y0 = (double)xy[1], x1 = (double)xy[2], y1 = (double)xy[3],
           x2 = (double)xy[4], y2 = (double)xy[5];
    // non-finite coordinates: the reference raises inside _bands (KN:54); we skip the triangle.
    if (!(isfinite(x0) && isfinite(y0) && isfinite(x1) && isfinite(y1) && isfinite(x2) && isfinite(y2)))
        return false;
    double area2 = xsub(xmul(xsub(x1, x0), xsub(y2, y0)), xmul(xsub(y1, y0), xsub(x2, x0)));  // KN:35
    if (area2 == 0.0) return false;                                                          // KN:36
    s.swapped = area2 < 0.0;                                                                 // KN:38
    if (s.swapped) { double tx = x1, ty = y1; x1 = x2; y1 = y2; x2 = tx; y2 = ty; }
    s.x0 = x0; s.y0 = y0; s.x1 = x1; s.y1 = y1; s.x2 = x2; s.y2 = y2;
    s.ax = xsub(x2, x1); s.ay = xsub(y2, y1);
    s.bx = xsub(x0, x2); s.by = xsub(y0, y2);
    s.cx = xsub(x1, x0); s.cy = xsub(y1, y0);
    s.t0 = s.ay < 0.0 || (s.ay == 0.0 && s.ax < 0.0);                                         // KN:75
    s.t1 = s.by < 0.0 || (s.by == 0.0 && s.bx < 0.0);                                         // KN:76
    s.t2 = s.cy < 0.0 || (s.cy == 0.0 && s.cx < 0.0);                                         // KN:77
    return true;
}

// Inclusive bbox of candidate texels.  Exact geometry needs only centres i+0.5 in [min, max],
// i.e. ceil(min-0.5) <= i <= floor(max-0.5).  The reference scans the wider box
// floor(min-0.5) .. ceil(max) (KN:54-57) and accepts whatever passes the ROUNDED edge tests, so a
// centre a few ulps outside the exact box could in principle still be accepted there.  A sign
// flip of a rounded edge function needs |e| <= ~4u*(|P|+|Q|), which bounds the distance of such
// a centre from the exact box by ~u * (triangle extent); the box below keeps
// a margin tol >= 2^-20 + 2^-30*max|coord| (ten orders of magnitude above that bound), clamped
// into the reference's box -- a subset of the reference's candidates that contains every texel
// the reference can accept.  Banding / bbox choice never changes a texel value (KN:23-24).
ML_DEV bool tri_bbox(TriSetup& s, long long width, long long height, long long row0, long long rows) {
    double xmin = fmin(fmin(s.x0, s.x1), s.x2), xmax = fmax(fmax(s.x0, s.x1), s.x2);
    double ymin = fmin(fmin(s.y0, s.y1), s.y2), ymax = fmax(fmax(s.y0, s.y1), s.y2);
    const double mabs = fmax(fmax(fabs(xmin), fabs(xmax)), fmax(fabs(ymin), fabs(ymax)));
    const double tol = 9.5367431640625e-07 + 9.313225746154785e-10 * mabs;
    double fx0 = fmax(ceil(xmin - 0.5 - tol), floor(xmin - 0.5));
    double fx1 = fmin(floor(xmax - 0.5 + tol), ceil(xmax));
    double fy0 = fmax(ceil(ymin - 0.5 - tol), floor(ymin - 0.5));
    double fy1 = fmin(floor(ymax - 0.5 + tol), ceil(ymax));
    double lox = 0.0, hix = (double)(width - 1);
    double loy = (double)row0, hiy = (double)(row0 + rows - 1);
    if (hiy > (double)(height - 1)) hiy = (double)(height - 1);
    if (fx0 < lox) fx0 = lox;
    if (fy0 < loy) fy0 = loy;
    if (fx1 > hix) fx1 = hix;
    if (fy1 > hiy) fy1 = hiy;
    if (fx1 < fx0 || fy1 < fy0) return false;
    s.ix0 = (int)fx0; s.ix1 = (int)fx1; s.iy0 = (int)fy0; s.iy1 = (int)fy1;
    return true;
}

// KN:68-81 at texel (x, y): edge functions at the centre (x+0.5, y+0.5) and the coverage test.
ML_DEV bool tri_inside(const TriSetup& s, int x, int y, double& e0, double& e1, double& e2) {
    const double cx = xadd((double)x, 0.5), cy = xadd((double)y, 0.5);       // KN:60, 63
    e0 = xsub(xmul(s.ax, xsub(cy, s.y1)), xmul(s.ay, xsub(cx, s.x1)));       // KN:72
    e1 = xsub(xmul(s.bx, xsub(cy, s.y2)), xmul(s.by, xsub(cx, s.x2)));       // KN:73
    e2 = xsub(xmul(s.cx, xsub(cy, s.y0)), xmul(s.cy, xsub(cx, s.x0)));       // KN:74
    const bool ok0 = (e0 > 0.0) || ((e0 == 0.0) && s.t0);                    // KN:78
    const bool ok1 = (e1 > 0.0) || ((e1 == 0.0) && s.t1);                    // KN:79
    const bool ok2 = (e2 > 0.0) || ((e2 == 0.0) && s.t2);                    // KN:80
    return ok0 && ok1 && ok2;
}

// ---------------------------------------------------------------------------------------------
// TEA fragment filters, KN:166-193, for one covered texel.
struct TeaParams {
    double ww, wh;          // window size (KN:179-181)
    double eps;             // depth bias
    double sfx, sfy, bx, by;
    const float* depth;     // [dh][dw] window depth plane, y-up rows
    const uint8_t* shape;   // [th][tw] tool shape plane
    long long dw, dh, tw, th;
    int eps_f32;            // 1: depth+eps rounded to float32 (numpy weak-scalar rule), 0: float64
};

// Filters after the clip-space interpolation: window KN:181, depth KN:185, tool range KN:189, shape
// KN:193.  The three last ones are independent tests ANDed together; they are evaluated in the
// order that lets the two dependent gathers (depth sample, shape sample) overlap each other and
// the zn division.  zc is passed in (KN:172 is computed by the caller from the same l's).
ML_DEV bool tea_filters(const TeaParams& p, double xc, double yc, double zc, double wc) {
    const double xn = xdiv(xc, wc), yn = xdiv(yc, wc);                            // KN:176-177
    const double xw = xmul(xmul(xadd(xn, 1.0), 0.5), p.ww);                       // KN:179
    const double yw = xmul(xmul(xadd(yn, 1.0), 0.5), p.wh);                       // KN:180
    if (!((xw >= 0.0) && (xw < p.ww) && (yw >= 0.0) && (yw < p.wh))) return false;    // KN:181
    const long long px = (long long)xw, py = (long long)yw;                       // KN:182-183
    const float dv = __ldg(p.depth + py * p.dw + px);
    const double s = xadd(xmul(p.sfx, xn), p.bx);                                 // KN:187
    const double t = xadd(xmul(p.sfy, yn), p.by);                                 // KN:188
    if (!((s >= 0.0) && (s <= 1.0) && (t >= 0.0) && (t <= 1.0))) return false;    // KN:189
    long long si = (long long)xmul(s, (double)p.tw), ti = (long long)xmul(t, (double)p.th);
    if (si > p.tw - 1) si = p.tw - 1;                                             // KN:191
    if (ti > p.th - 1) ti = p.th - 1;                                             // KN:192
    const uint8_t sh = __ldg(p.shape + ti * p.tw + si);                           // KN:193
    const double zn = xdiv(zc, wc);                                               // KN:178
    const double df = xmul(xadd(zn, 1.0), 0.5);                                   // KN:184
    const double lim = p.eps_f32 ? (double)__fadd_rn(dv, (float)p.eps) : xadd((double)dv, p.eps);
    return (df <= lim) && (sh != 0);                                              // KN:185, 193
}

ML_DEV bool tea_fragment(const TeaParams& p, double e0, double e1, double e2,
                         const double* __restrict__ c0, const double* __restrict__ c1,
                         const double* __restrict__ c2) {
    const double esum = xadd(xadd(e0, e1), e2);                                   // KN:166
    const double l0 = xdiv(e0, esum), l1 = xdiv(e1, esum), l2 = xdiv(e2, esum);   // KN:167-169
    const double wc = xadd(xadd(xmul(l0, c0[3]), xmul(l1, c1[3])), xmul(l2, c2[3]));  // KN:173
    if (!(wc > 0.0)) return false;                                                // KN:174
    const double xc = xadd(xadd(xmul(l0, c0[0]), xmul(l1, c1[0])), xmul(l2, c2[0]));  // KN:170
    const double yc = xadd(xadd(xmul(l0, c0[1]), xmul(l1, c1[1])), xmul(l2, c2[1]));  // KN:171
    const double zc = xadd(xadd(xmul(l0, c0[2]), xmul(l1, c1[2])), xmul(l2, c2[2]));  // KN:172
    return tea_filters(p, xc, yc, zc, wc);
}
