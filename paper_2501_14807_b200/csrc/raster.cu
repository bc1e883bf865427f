// Texture-space rasteriser for sm_100a: coverage_fill, raster_depth, raster_tea (direct,
// per-triangle) and the triangle-id pass of the surface map.
//
// Reference semantics: pkg/src/meshlayers/_kernels_numpy.py (KN) 84-100, 103-132, 135-203.
// The reference walks triangles serially and each triangle's bbox with numpy array ops; here
// every (triangle, texel) pair is an independent work item, which is legal because
//   * coverage / TEA planes and counts do not depend on triangle order,
//   * the depth plane equals min(initial, min_t float32(d_t)) for any order.
//
// Work distribution (B200: 148 SMs, thousands of resident warps):
//   pass A  one WARP per triangle: per-row covered spans by bisection on the exact edge predicate,
//           then the covered texels are enumerated 32 at a time (see raster_warp_kernel).  Triangles
//           whose bbox exceeds SMALL_MAX texels are not rasterised here but appended to a
//           "large" list together with their number of CHUNK-texel chunks.
//   pass B  single-block exclusive scan of the chunk counts.
//   pass C  one BLOCK per (large triangle, chunk): a fixed grid strides over the scanned
//           work-item range, finds its triangle by binary search, and covers CHUNK
//           consecutive bbox texels.  No host synchronisation anywhere.
#include "common.cuh"
#include "meshlayers_b200.h"
#include "internal.h"

namespace {

constexpr int SMALL_MAX = 1024;       // bbox texels handled by one warp
constexpr int CHUNK = 2048;           // bbox texels per block work item (large triangles)
constexpr int BLOCK = 256;

struct LargeList {
    int* tri;                         // [ntri] triangle indices
    unsigned long long* off;          // [ntri+1] chunk counts, then exclusive offsets
    unsigned long long* count;        // number of large triangles
    unsigned long long* total;        // total chunks (written by the scan)
};

// ------------------------------------------------------------------ fragment functors
// Each functor provides:
//   struct Tri;  Tri setup(long long t, const TriSetup&)       per-triangle attribute fetch
//   void fragment(const Tri&, long long t, int x, int y, e0,e1,e2, long long& c0, long long& c1)
// Planes are slab-local: texel (x, y) lives at (y - row0) * width + x.

struct CoverageFn {
    static constexpr bool NEEDS_E = false;        // fragment() ignores the edge-function values
    static constexpr bool WORD_SPANS = true;      // spans are written word by word (span_words below)
    uint8_t* out; long long width, row0;
    struct Tri {};
    // Set the bytes `ones` (0x01 in every byte lane to set) of one aligned 32-bit word with ONE atomic
    // and count the lanes that were 0 (KN:97-99 for up to four texels).  A lane that held some other
    // non-zero value is forced to exactly 1 afterwards (byte_set1_was0), which cannot change the count.
    ML_DEV uintptr_t row_address(int y) const { return (uintptr_t)(out + (y - row0) * width); }
    ML_DEV void word_fragment(uint32_t* word, uint32_t ones, long long& c0) const {
        const uint32_t old = atomicOr(word, ones);
        const uint32_t lanes = ones * 0x80u;                          // bit 7 of every byte lane to set
        c0 += __popc(zero_bytes_msb(old) & lanes);
        uint32_t odd = (old & ~0x01010101u) & (ones * 0xffu);         // lanes holding neither 0 nor 1
        while (odd) {
            const int b = (__ffs(odd) - 1) >> 3;
            odd &= ~(0xffu << (8 * b));
            byte_set1_was0((uint8_t*)word, b);
        }
    }
    ML_DEV Tri setup(long long, const TriSetup&) const { return Tri(); }
    ML_DEV void fragment(const Tri&, long long, int x, int y, double, double, double,
                         long long& c0, long long&) const {
        if (byte_set1_was0(out, (y - row0) * width + x)) ++c0;           // KN:97-99
    }
};

struct TriIdFn {
    static constexpr bool NEEDS_E = false;
    static constexpr bool WORD_SPANS = false;
    int* tri_id; long long width, row0;
    struct Tri {};
    ML_DEV Tri setup(long long, const TriSetup&) const { return Tri(); }
    ML_DEV void fragment(const Tri&, long long t, int x, int y, double, double, double,
                         long long& c0, long long&) const {
        // last triangle in submission order owns the texel.  The old value is not
        // used, so this is a fire-and-forget reduction (RED.MAX): no lane waits for the L2 round trip.
        // Overlap events = fragments - covered texels; the resolve pass counts the covered ones.
        atomicMax(tri_id + (y - row0) * width + x, (int)t);
        ++c0;                               // fragments
    }
};

template <typename T>
struct DepthFn {
    static constexpr bool NEEDS_E = true;
    static constexpr bool WORD_SPANS = false;
    const T* tri_zn; float* depth; long long width;
    struct Tri { double z0, z1, z2; };
    ML_DEV Tri setup(long long t, const TriSetup& s) const {
        Tri r;
        r.z0 = (double)tri_zn[3 * t];
        r.z1 = (double)tri_zn[3 * t + (s.swapped ? 2 : 1)];              // KN:40 swap attrs too
        r.z2 = (double)tri_zn[3 * t + (s.swapped ? 1 : 2)];
        return r;
    }
    ML_DEV void fragment(const Tri& a, long long, int x, int y, double e0, double e1, double e2,
                         long long&, long long&) const {
        const double esum = xadd(xadd(e0, e1), e2);                                   // KN:122
        const double l0 = xdiv(e0, esum), l1 = xdiv(e1, esum), l2 = xdiv(e2, esum);   // KN:123-125
        const double znf = xadd(xadd(xmul(l0, a.z0), xmul(l1, a.z1)), xmul(l2, a.z2));  // KN:126
        const double d = xmul(xadd(znf, 1.0), 0.5);                                   // KN:127
        // sequential rule "if d < s: s = f32(d)" (KN:129-130) == running minimum in float32
        // (monotone rounding): CAS loop keeps exact IEEE compare semantics.
        float* p = depth + (long long)y * width + x;
        const float fd = (float)d;
        float cur = *(volatile float*)p;
        while (d < (double)cur) {
            const int assumed = __float_as_int(cur);
            const int old = atomicCAS((int*)p, assumed, __float_as_int(fd));
            if (old == assumed) break;
            cur = __int_as_float(old);
        }
    }
};

template <typename T>
struct TeaFn {
    static constexpr bool NEEDS_E = true;
    static constexpr bool WORD_SPANS = false;
    const T* tri_clip; TeaParams p;
    void* data; uint8_t* mask; uint8_t* edited;
    long long width, row0; uint32_t value; int esize;
    const uint32_t* flags;            // ml_tea_classify bitmap of this stroke (NULL: evaluate everything)
    struct Tri { double c0[4], c1[4], c2[4]; bool keep; };
    ML_DEV Tri setup(long long t, const TriSetup& s) const {
        Tri r;
        // a triangle the classification pass proved unreachable only counts its fragments (KN:158-161)
        r.keep = flags ? ((flags[t >> 5] >> (t & 31)) & 1u) != 0 : true;
        if (!r.keep) return r;
        const T* c = tri_clip + 12 * t;
        const int i1 = s.swapped ? 8 : 4, i2 = s.swapped ? 4 : 8;        // KN:40 swap attrs too
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            r.c0[k] = (double)c[k]; r.c1[k] = (double)c[i1 + k]; r.c2[k] = (double)c[i2 + k];
        }
        return r;
    }
    ML_DEV void fragment(const Tri& a, long long, int x, int y, double e0, double e1, double e2,
                         long long& c0, long long& c1) const {
        ++c1;                                                            // fragments, KN:158-161
        if (!a.keep || !tea_fragment(p, e0, e1, e2, a.c0, a.c1, a.c2)) return;
        const long long i = (y - row0) * width + x;
        if (byte_set1_was0(edited, i)) ++c0;                             // KN:198-199, 202
        if (data) store_value(data, esize, i, value);                    // KN:200 (NULL: the caller only wants the hit set)
        if (mask) mask[i] = 1;                                           // KN:201
    }
};

// ------------------------------------------------------------------ pass A
// Row spans.  For a fixed row the edge function e_i(x) = fl(K_i - fl(m_i * fl(cx - xo_i))) is a
// MONOTONE function of the column (floating-point subtraction, multiplication by a constant and
// rounding are all monotone), so the accepted columns of each edge form a prefix (m_i > 0), a suffix
// (m_i < 0) or everything / nothing (m_i == 0), and the covered texels of the row are one interval.
// Its ends are found by bisection on the EXACT predicate of KN:72-80 -- no analytic intersection, so
// the covered set is bit-for-bit the one the per-texel test gives -- in O(log w) probes per edge.
struct RowEdge { double K, m, xo; bool tie; };            // e(x) = K - m * ((x + 0.5) - xo)
ML_DEV bool edge_accepts(const RowEdge& g, int x) {
    const double e = xsub(g.K, xmul(g.m, xsub(xadd((double)x, 0.5), g.xo)));
    return (e > 0.0) || ((e == 0.0) && g.tie);                                   // KN:78-80
}
// clip [xa, xb] to the columns edge g accepts
ML_DEV void edge_clip(const RowEdge& g, int& xa, int& xb) {
    if (xa > xb) return;
    if (g.m == 0.0) { if (!edge_accepts(g, xa)) xb = xa - 1; return; }
    if (g.m > 0.0) {                       // non-increasing in x: accepted columns are a prefix
        if (!edge_accepts(g, xa)) { xb = xa - 1; return; }
        int lo = xa, hi = xb;              // invariant: lo accepted; answer = last accepted in [lo, hi]
        while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (edge_accepts(g, mid)) lo = mid; else hi = mid - 1; }
        xb = lo;
    } else {                               // non-decreasing: accepted columns are a suffix
        if (!edge_accepts(g, xb)) { xb = xa - 1; return; }
        int lo = xa, hi = xb;              // invariant: hi accepted; answer = first accepted in [lo, hi]
        while (lo < hi) { const int mid = (lo + hi) >> 1; if (edge_accepts(g, mid)) hi = mid; else lo = mid + 1; }
        xa = hi;
    }
}
// covered interval of row y (empty: xa > xb)
ML_DEV void row_span(const TriSetup& s, int y, int& xa, int& xb) {
    const double cy = xadd((double)y, 0.5);                                      // KN:63
    xa = s.ix0; xb = s.ix1;
    edge_clip(RowEdge{xmul(s.ax, xsub(cy, s.y1)), s.ay, s.x1, s.t0}, xa, xb);    // KN:72
    edge_clip(RowEdge{xmul(s.bx, xsub(cy, s.y2)), s.by, s.x2, s.t1}, xa, xb);    // KN:73
    edge_clip(RowEdge{xmul(s.cx, xsub(cy, s.y0)), s.cy, s.x0, s.t2}, xa, xb);    // KN:74
}

// One WARP per triangle.  Tiny boxes (<= 32 texels) are tested texel by texel in one step.  Larger
// ones: (1) lane r finds the span of row r by bisection, (2) a warp prefix sum over the span lengths
// enumerates the covered texels, (3) lanes take them 32 at a time in row-major order (neighbouring
// lanes on neighbouring texels), so no lane is spent on an uncovered texel of the box.
// SPANS = false keeps only the texel-by-texel walk (lanes stride over the box): the leaner kernel for
// inputs whose triangles cover a few texels each (depth pass, coarse atlases); the host picks the
// variant from the average texels per triangle -- both give identical results for any input.
template <typename T, typename F, bool SPANS>
__global__ void __launch_bounds__(BLOCK)
raster_warp_kernel(const T* __restrict__ tri_xy, long long ntri, long long width, long long height,
                   long long row0, long long rows, F f, LargeList ll,
                   unsigned long long* counters, const int* __restrict__ slab_list,
                   const unsigned long long* __restrict__ slab_count) {
    const int lane = threadIdx.x & 31;
    const long long nwarps = (long long)gridDim.x * (BLOCK / 32);
    long long c0 = 0, c1 = 0;
    // row slabs: walk the slab's triangle list (ml_slab_triangle_list) instead of every triangle of the mesh
    const long long nwork = slab_list ? (long long)*slab_count : ntri;
    for (long long k = (long long)blockIdx.x * (BLOCK / 32) + (threadIdx.x >> 5); k < nwork; k += nwarps) {
        const long long t = slab_list ? (long long)slab_list[k] : k;
        TriSetup s;
        if (!tri_load_ccw(tri_xy + 6 * t, s)) continue;
        if (!tri_bbox(s, width, height, row0, rows)) continue;
        const int bw = s.ix1 - s.ix0 + 1, bh = s.iy1 - s.iy0 + 1;
        const long long n = (long long)bw * bh;
        if (n > SMALL_MAX) {
            if (lane == 0) {
                unsigned long long k = atomicAdd(ll.count, 1ull);
                ll.tri[k] = (int)t;
                ll.off[k] = (unsigned long long)((n + CHUNK - 1) / CHUNK);
            }
            continue;
        }
        const typename F::Tri a = f.setup(t, s);
        if (!SPANS || n <= 64) {
            for (int j = lane; j < (int)n; j += 32) {
                const int yy = j / bw, x = s.ix0 + (j - yy * bw), y = s.iy0 + yy;
                double e0, e1, e2;
                if (tri_inside(s, x, y, e0, e1, e2)) f.fragment(a, t, x, y, e0, e1, e2, c0, c1);
            }
            continue;
        }
        for (int rb = 0; rb < bh; rb += 32) {
            int xa = 1, xb = 0;
            if (rb + lane < bh) row_span(s, s.iy0 + rb + lane, xa, xb);
            // items to enumerate: covered texels, or (byte planes) the aligned 32-bit words they occupy
            int len = xb >= xa ? xb - xa + 1 : 0, mis = 0;
            if constexpr (F::WORD_SPANS) {
                mis = (int)(f.row_address(s.iy0 + rb + lane) & 3);        // misalignment of the row start
                if (len) len = ((mis + xb) >> 2) - ((mis + xa) >> 2) + 1;
            }
            int pre = len;                                   // inclusive prefix sum of the item counts
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) { const int v = __shfl_up_sync(0xffffffffu, pre, o); if (lane >= o) pre += v; }
            const int total = __shfl_sync(0xffffffffu, pre, 31);
            const int excl = pre - len;
#pragma unroll 2
            for (int kb = 0; kb < total; kb += 32) {
                const int k = kb + lane;
                int lo = 0, hi = 31;                         // first lane whose inclusive prefix exceeds k
#pragma unroll
                for (int step = 0; step < 5; ++step) {
                    const int mid = (lo + hi) >> 1;
                    const int pm = __shfl_sync(0xffffffffu, pre, mid);
                    if (k < pm) hi = mid; else lo = mid + 1;
                }
                const int r = lo & 31;
                const int ex = __shfl_sync(0xffffffffu, excl, r), xs = __shfl_sync(0xffffffffu, xa, r);
                if constexpr (F::WORD_SPANS) {
                    const int xe = __shfl_sync(0xffffffffu, xb, r), ms = __shfl_sync(0xffffffffu, mis, r);
                    if (k < total) {
                        const int w = ((ms + xs) >> 2) + (k - ex);            // word of the row, from its aligned base
                        const int b0 = max(ms + xs - 4 * w, 0), b1 = min(ms + xe - 4 * w, 3);   // byte lanes b0..b1
                        const uint32_t ones = 0x01010101u & (0xffffffffu >> (8 * (3 - b1))) & (0xffffffffu << (8 * b0));
                        f.word_fragment((uint32_t*)(f.row_address(s.iy0 + rb + r) - ms) + w, ones, c0);
                    }
                    continue;
                }
                if (k < total) {
                    const int x = xs + (k - ex), y = s.iy0 + rb + r;
                    double e0 = 0.0, e1 = 0.0, e2 = 0.0;
                    if (F::NEEDS_E) tri_inside(s, x, y, e0, e1, e2);             // barycentric numerators, KN:72-74
                    f.fragment(a, t, x, y, e0, e1, e2, c0, c1);
                }
            }
        }
    }
    block_count_add(c0, counters);
    block_count_add(c1, counters + 1);
}

// ------------------------------------------------------------------ pass B
// In-place exclusive scan of off[0..count) by one block; writes off[count] = total as well.
__global__ void __launch_bounds__(1024) scan_kernel(LargeList ll) {
    __shared__ unsigned long long s_sum[1024];
    const unsigned long long n = *ll.count;
    const unsigned long long per = (n + 1023) / 1024;
    const unsigned long long b = threadIdx.x * per, e = (b + per < n) ? b + per : n;
    unsigned long long acc = 0;
    for (unsigned long long i = b; i < e; ++i) acc += ll.off[i];
    s_sum[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {                 // Hillis-Steele inclusive scan
        unsigned long long v = (threadIdx.x >= o) ? s_sum[threadIdx.x - o] : 0;
        __syncthreads();
        s_sum[threadIdx.x] += v;
        __syncthreads();
    }
    unsigned long long run = s_sum[threadIdx.x] - acc;   // exclusive prefix of this thread
    for (unsigned long long i = b; i < e; ++i) { unsigned long long c = ll.off[i]; ll.off[i] = run; run += c; }
    if (threadIdx.x == 1023) { ll.off[n] = s_sum[1023]; *ll.total = s_sum[1023]; }
}

// ------------------------------------------------------------------ pass C
template <typename T, typename F>
__global__ void __launch_bounds__(BLOCK)
raster_chunk_kernel(const T* __restrict__ tri_xy, long long width, long long height,
                    long long row0, long long rows, F f, LargeList ll,
                    unsigned long long* counters) {
    __shared__ long long s_k;
    const unsigned long long total = *ll.total, nl = *ll.count;
    long long c0 = 0, c1 = 0;
    for (unsigned long long w = blockIdx.x; w < total; w += gridDim.x) {
        if (threadIdx.x == 0) {                          // largest k with off[k] <= w
            unsigned long long lo = 0, hi = nl;
            while (hi - lo > 1) { unsigned long long mid = (lo + hi) >> 1; if (ll.off[mid] <= w) lo = mid; else hi = mid; }
            s_k = (long long)lo;
        }
        __syncthreads();
        const long long k = s_k;
        __syncthreads();
        const long long t = ll.tri[k];
        TriSetup s;
        tri_load_ccw(tri_xy + 6 * t, s);
        tri_bbox(s, width, height, row0, rows);
        const long long bw = s.ix1 - s.ix0 + 1, bh = s.iy1 - s.iy0 + 1, n = bw * bh;
        const long long j0 = (long long)(w - ll.off[k]) * CHUNK;
        const long long j1 = (j0 + CHUNK < n) ? j0 + CHUNK : n;
        const typename F::Tri a = f.setup(t, s);
        for (long long j = j0 + threadIdx.x; j < j1; j += BLOCK) {
            const long long yy = j / bw;
            const int x = s.ix0 + (int)(j - yy * bw), y = s.iy0 + (int)yy;
            double e0, e1, e2;
            if (tri_inside(s, x, y, e0, e1, e2)) f.fragment(a, t, x, y, e0, e1, e2, c0, c1);
        }
    }
    block_count_add(c0, counters);
    block_count_add(c1, counters + 1);
}

// SPEC.md:129-137 ``rasterize`` with a per-triangle output value: after the owner pass (last triangle
// in submission order wins) every covered texel takes its owner's value unless the rule
// discarded that triangle.  4 texels per thread (128-bit id load), 1 / 2 / 4-byte elements.
template <typename E>
__global__ void __launch_bounds__(BLOCK)
owner_values_kernel(const int* __restrict__ tri_id, long long n, const E* __restrict__ values,
                    const uint8_t* __restrict__ keep, E* __restrict__ out, unsigned long long* written) {
    long long cnt = 0;
    const long long nthreads = (long long)gridDim.x * BLOCK;
    for (long long i = (long long)blockIdx.x * BLOCK + threadIdx.x; i < n; i += nthreads) {
        const int t = tri_id[i];
        if (t < 0 || (keep && keep[t] == 0)) continue;
        out[i] = values[t];
        ++cnt;
    }
    block_count_add(cnt, written);
}

// Row-slab triangle list: one thread per triangle, the reference's own conservative row range
// floor(ymin - 0.5) .. ceil(ymax) (KN:54-57; tri_bbox never looks outside it), ballot-compacted.
template <typename T>
__global__ void __launch_bounds__(BLOCK)
slab_list_kernel(const T* __restrict__ tri_xy, long long ntri, long long row0, long long rows,
                 int* __restrict__ list, unsigned long long* count) {
    const int lane = threadIdx.x & 31;
    for (long long t0 = (long long)blockIdx.x * BLOCK; t0 < ntri; t0 += (long long)gridDim.x * BLOCK) {
        const long long t = t0 + threadIdx.x;
        bool keep = false;
        if (t < ntri) {
            const double y0 = (double)tri_xy[6 * t + 1], y1 = (double)tri_xy[6 * t + 3], y2 = (double)tri_xy[6 * t + 5];
            const double lo = floor(fmin(fmin(y0, y1), y2) - 0.5), hi = ceil(fmax(fmax(y0, y1), y2));
            keep = hi >= (double)row0 && lo <= (double)(row0 + rows - 1);      // false for NaN rows: such triangles are skipped anyway
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (!bal) continue;
        unsigned long long slot = 0;
        if (lane == 0) slot = atomicAdd(count, (unsigned long long)__popc(bal));
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (keep) list[slot + __popc(bal & ((1u << lane) - 1u))] = (int)t;
    }
}

}  // namespace

int ml_slab_triangle_list(const void* tri_xy, int tri_dtype, long long ntri, long long row0, long long rows,
                          int* list, unsigned long long* count, cudaStream_t st) {
    if (ntri <= 0) return ML_OK;
    long long blocks = (ntri + BLOCK - 1) / BLOCK;
    const long long cap = (long long)ml_sm_count() * 16;
    if (blocks > cap) blocks = cap;
    if (tri_dtype == ML_F32) slab_list_kernel<float><<<(unsigned)blocks, BLOCK, 0, st>>>((const float*)tri_xy, ntri, row0, rows, list, count);
    else slab_list_kernel<double><<<(unsigned)blocks, BLOCK, 0, st>>>((const double*)tri_xy, ntri, row0, rows, list, count);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

namespace {

template <typename T, typename F>
int raster_launch(const T* tri_xy, long long ntri, long long width, long long height,
                  long long row0, long long rows, const F& f, void* workspace, size_t ws_bytes,
                  unsigned long long* counters, cudaStream_t st) {
    if (ntri <= 0 || rows <= 0 || width <= 0) return ML_OK;
    if (ntri > 0x7fffffffLL) return ml_fail(ML_ERR_ARG, "more than 2^31-1 triangles");
    if (ws_bytes < ml_raster_workspace_bytes(ntri)) return ml_fail(ML_ERR_ARG, "raster workspace too small");
    // workspace layout: [count, total, c0, c1, slab count, -] u64 | off[ntri+1] u64 | tri[ntri] i32 | TEA flags | slab list[ntri] i32
    unsigned long long* head = (unsigned long long*)workspace;
    LargeList ll;
    ll.count = head; ll.total = head + 1;
    ll.off = head + 6;
    ll.tri = (int*)(ll.off + ntri + 1);
    unsigned long long* ctr = counters ? counters : head + 2;
    ML_CUDA(cudaMemsetAsync(head, 0, 6 * sizeof(unsigned long long), st));
    const int* slab_list = nullptr;
    const unsigned long long* slab_count = nullptr;
    if (ml_slab_uses_list(rows, height, ntri)) {
        int* list = (int*)((char*)workspace + ml_raster_workspace_bytes(ntri) - (size_t)ntri * sizeof(int) - 16);
        const int rc = ml_slab_triangle_list(tri_xy, sizeof(T) == 4 ? ML_F32 : ML_F64, ntri, row0, rows, list, head + 4, st);
        if (rc != ML_OK) return rc;
        slab_list = list; slab_count = head + 4;
    }
    const long long warps_per_block = BLOCK / 32;
    long long blocks = (ntri + warps_per_block - 1) / warps_per_block;
    const long long cap = (long long)ml_sm_count() * 64;
    if (blocks > cap) blocks = cap;
    if ((double)width * (double)rows >= 40.0 * (double)ntri)          // >= ~40 texels per triangle: row spans pay off
        raster_warp_kernel<T, F, true><<<(unsigned)blocks, BLOCK, 0, st>>>(tri_xy, ntri, width, height, row0, rows, f, ll, ctr, slab_list, slab_count);
    else
        raster_warp_kernel<T, F, false><<<(unsigned)blocks, BLOCK, 0, st>>>(tri_xy, ntri, width, height, row0, rows, f, ll, ctr, slab_list, slab_count);
    scan_kernel<<<1, 1024, 0, st>>>(ll);
    raster_chunk_kernel<T, F><<<(unsigned)(ml_sm_count() * 8), BLOCK, 0, st>>>(tri_xy, width, height, row0, rows, f, ll, ctr);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

}  // namespace

extern "C" {

size_t ml_raster_workspace_bytes(int64_t ntri) {
    if (ntri < 0) ntri = 0;
    size_t b = 6 * sizeof(unsigned long long) + (size_t)(ntri + 1) * sizeof(unsigned long long) +
               (size_t)ntri * sizeof(int) + (size_t)((ntri + 31) / 32) * sizeof(uint32_t) + 64;   // + TEA triangle flags
    b = (b + 15) & ~(size_t)15;
    return b + (size_t)ntri * sizeof(int) + 16;                                                  // + row-slab triangle list (last)
}

int ml_coverage_fill(const void* tri_xy, int tri_dtype, int64_t ntri, int64_t width, int64_t height,
                     int64_t row0, int64_t rows, uint8_t* out, uint64_t* written,
                     void* workspace, size_t workspace_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    CoverageFn f{out, width, row0};
    unsigned long long* ctr = (unsigned long long*)written;
    if (tri_dtype == ML_F32)
        return raster_launch((const float*)tri_xy, ntri, width, height, row0, rows, f, workspace, workspace_bytes, ctr, st);
    if (tri_dtype == ML_F64)
        return raster_launch((const double*)tri_xy, ntri, width, height, row0, rows, f, workspace, workspace_bytes, ctr, st);
    return ml_fail(ML_ERR_ARG, "tri_dtype must be ML_F32 or ML_F64");
}

int ml_raster_tri_id(const void* tri_xy, int tri_dtype, int64_t ntri, int64_t width, int64_t height,
                     int64_t row0, int64_t rows, int32_t* tri_id, uint64_t* counters,
                     void* workspace, size_t workspace_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (rows > 0 && width > 0)
        ML_CUDA(cudaMemsetAsync(tri_id, 0xff, (size_t)rows * width * sizeof(int32_t), st));   // -1
    TriIdFn f{tri_id, width, row0};
    unsigned long long* ctr = (unsigned long long*)counters;
    if (tri_dtype == ML_F32)
        return raster_launch((const float*)tri_xy, ntri, width, height, row0, rows, f, workspace, workspace_bytes, ctr, st);
    if (tri_dtype == ML_F64)
        return raster_launch((const double*)tri_xy, ntri, width, height, row0, rows, f, workspace, workspace_bytes, ctr, st);
    return ml_fail(ML_ERR_ARG, "tri_dtype must be ML_F32 or ML_F64");
}

int ml_owner_values(const int32_t* tri_id, int64_t n, const void* values, const uint8_t* keep, int esize,
                    void* out, uint64_t* written, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) return ML_OK;
    long long blocks = (n + BLOCK - 1) / BLOCK;
    const long long cap = (long long)ml_sm_count() * 32;
    if (blocks > cap) blocks = cap;
    unsigned long long* w = (unsigned long long*)written;
    if (esize == 1) owner_values_kernel<uint8_t><<<(unsigned)blocks, BLOCK, 0, st>>>(tri_id, n, (const uint8_t*)values, keep, (uint8_t*)out, w);
    else if (esize == 2) owner_values_kernel<uint16_t><<<(unsigned)blocks, BLOCK, 0, st>>>(tri_id, n, (const uint16_t*)values, keep, (uint16_t*)out, w);
    else if (esize == 4) owner_values_kernel<uint32_t><<<(unsigned)blocks, BLOCK, 0, st>>>(tri_id, n, (const uint32_t*)values, keep, (uint32_t*)out, w);
    else return ml_fail(ML_ERR_ARG, "esize must be 1, 2 or 4");
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int ml_raster_depth(const void* tri_xy, const void* tri_zn, int tri_dtype, int64_t ntri,
                    float* depth, int64_t width, int64_t height,
                    void* workspace, size_t workspace_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (tri_dtype == ML_F32) {
        DepthFn<float> f{(const float*)tri_zn, depth, width};
        return raster_launch((const float*)tri_xy, ntri, width, height, 0, height, f, workspace, workspace_bytes, nullptr, st);
    }
    if (tri_dtype == ML_F64) {
        DepthFn<double> f{(const double*)tri_zn, depth, width};
        return raster_launch((const double*)tri_xy, ntri, width, height, 0, height, f, workspace, workspace_bytes, nullptr, st);
    }
    return ml_fail(ML_ERR_ARG, "tri_dtype must be ML_F32 or ML_F64");
}

int ml_raster_tea(const void* tri_xy, const void* tri_clip, int tri_dtype, int64_t ntri,
                  int64_t width, int64_t height, int64_t row0, int64_t rows,
                  const ml_tea_params* tp, void* data, int esize, uint32_t value_bits,
                  uint8_t* mask, uint8_t* edited, uint64_t* counters,
                  void* workspace, size_t workspace_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (esize != 1 && esize != 2 && esize != 4) return ml_fail(ML_ERR_ARG, "esize must be 1, 2 or 4");
    TeaParams p = ml_make_tea_params(tp);
    unsigned long long* ctr = (unsigned long long*)counters;
    // per-stroke triangle classification (surface.cu): triangles that provably cannot pass the
    // w > 0 / window / tool-range filters skip the float64 evaluation; their fragments are still
    // rasterised and counted, so planes and both counts are unchanged
    uint32_t* flags = nullptr;
    if (ntri > 0 && workspace && workspace_bytes >= ml_raster_workspace_bytes(ntri) && (tri_dtype == ML_F32 || tri_dtype == ML_F64)) {
        flags = (uint32_t*)((char*)workspace + 6 * sizeof(unsigned long long) + (size_t)(ntri + 1) * sizeof(unsigned long long) +
                            (size_t)ntri * sizeof(int));
        const int rc = ml_tea_classify(tri_clip, tri_dtype, ntri, tp, flags, nullptr, width, height, row0, rows, nullptr, stream);
        if (rc != ML_OK) return rc;
    }
    if (tri_dtype == ML_F32) {
        TeaFn<float> f{(const float*)tri_clip, p, data, mask, edited, width, row0, value_bits, esize, flags};
        return raster_launch((const float*)tri_xy, ntri, width, height, row0, rows, f, workspace, workspace_bytes, ctr, st);
    }
    if (tri_dtype == ML_F64) {
        TeaFn<double> f{(const double*)tri_clip, p, data, mask, edited, width, row0, value_bits, esize, flags};
        return raster_launch((const double*)tri_xy, ntri, width, height, row0, rows, f, workspace, workspace_bytes, ctr, st);
    }
    return ml_fail(ML_ERR_ARG, "tri_dtype must be ML_F32 or ML_F64");
}

}  // extern "C"
