// Per-layer area / statistics reductions (north star (4)).  No reference code beyond
// mesh_surface_area and the precision metric; the frozen
// definitions are oracle/kn_port.c ext_layer_area / ext_label_area / ext_layer_stats.
//
// ml_layer_area: one pass reads the float32 area plane once plus G <= 8 mask planes per launch
// group (4 + G B/texel), accumulates in float64 registers, reduces with warp shuffles and issues
// ONE float64 atomic per block per layer.
#include <stdlib.h>
#include <string.h>
#include "common.cuh"
#include "bulk.cuh"
#include "meshlayers_b200.h"
#include "internal.h"

namespace {

constexpr int BLOCK = 256;
constexpr int MAX_G = 8;

constexpr int MAX_PEERS = 16;

struct AreaArgs {
    const uint8_t* mask[MAX_G];
    double* sums;              // [G] slice of the caller's array
    unsigned long long* counts;
    // Fused cross-rank reduction (row-sharded atlases): npeers > 0 -> every block adds its partial sums with
    // SYSTEM-scope atomics into the same slots of EVERY rank's result row (peer memory over NVLink, IPC-mapped;
    // own row included), so the all-reduce of the areas happens inside the reduction kernel.
    int npeers;
    double* peer_sums[MAX_PEERS];
    unsigned long long* peer_counts[MAX_PEERS];
};

// one value per block and layer: to the local accumulator, or to the row of every rank
ML_DEV void area_emit(const AreaArgs& a, int g, double t, unsigned long long c, bool lane0) {
    if (!lane0) return;
    if (a.npeers == 0) {
        if (t != 0.0) atomicAdd(a.sums + g, t);
        if (a.counts && c) atomicAdd(a.counts + g, c);
        return;
    }
    for (int p = 0; p < a.npeers; ++p) {
        if (t != 0.0) atomicAdd_system(a.peer_sums[p] + g, t);
        if (c) atomicAdd_system(a.peer_counts[p] + g, c);
    }
}

// block reduction of (acc, cnt) per layer over NW warps + area_emit by one thread
template <int G, int NW>
ML_DEV void area_commit(const AreaArgs& a, const double (&acc)[G], const unsigned (&cnt)[G]) {
    __shared__ double s_sum[NW];
    __shared__ unsigned long long s_cnt[NW];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const double v = warp_sum(acc[g]);
        const long long c = warp_sum((long long)cnt[g]);
        if (lane == 0) { s_sum[wid] = v; s_cnt[wid] = (unsigned long long)c; }
        __syncthreads();
        if (wid == 0) {
            double t = lane < NW ? s_sum[lane] : 0.0;
            long long tc = lane < NW ? (long long)s_cnt[lane] : 0;
            t = warp_sum(t);
            tc = warp_sum(tc);
            area_emit(a, g, t, (unsigned long long)tc, lane == 0);
        }
        __syncthreads();
    }
}

ML_DEV void block_sum_atomic(double v, double* out) {
    __shared__ double s_part[BLOCK / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) s_part[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double t = lane < BLOCK / 32 ? s_part[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0 && t != 0.0) atomicAdd(out, t);
    }
    __syncthreads();
}

// 16 texels per thread step: four 128-bit area loads + one 128-bit load per mask plane.
template <int G, bool VECTOR>
__global__ void __launch_bounds__(BLOCK, 2)
area_kernel(const float* __restrict__ area, AreaArgs a, long long n) {
    double acc[G];
    unsigned cnt[G];                      // per-thread texel counts (< 2^32 texels per thread)
#pragma unroll
    for (int g = 0; g < G; ++g) { acc[g] = 0.0; cnt[g] = 0; }
    const long long tid = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * BLOCK;
    long long done = 0;
    if (VECTOR) {
        // Layer masks are spatially coherent and mostly empty, so the area vector of a 16-texel step is
        // fetched only when some mask of the group has a texel in it.  That makes the area load depend
        // on the mask loads; the dependency is hidden by requesting the masks of the thread's NEXT step
        // before the area of the current one (software pipelining), so the bytes in flight stay those of
        // an unconditional stream.  Most vectors lie entirely outside or entirely inside a layer (mask
        // bytes written by this library are exactly 0 / 1): whole 4-texel words are skipped or added as
        // one pre-summed double; only words on a mask boundary, or masks using other non-zero byte
        // values, take the per-texel path.  Summation order is free (1e-6 relative, north star).
        const long long nv = n >> 4;
        uint4 mn[G];
        if (tid < nv) {
#pragma unroll
            for (int g = 0; g < G; ++g) mn[g] = ld_stream((const uint4*)a.mask[g] + tid);
        }
        for (long long v = tid; v < nv; v += nthreads) {
            uint4 m[G];
#pragma unroll
            for (int g = 0; g < G; ++g) m[g] = mn[g];
            if (v + nthreads < nv) {
#pragma unroll
                for (int g = 0; g < G; ++g) mn[g] = ld_stream((const uint4*)a.mask[g] + v + nthreads);
            }
            uint32_t anyset = 0;
#pragma unroll
            for (int g = 0; g < G; ++g) anyset |= m[g].x | m[g].y | m[g].z | m[g].w;
            if (anyset == 0) continue;
            float4 ar[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) ar[j] = ld_stream((const float4*)area + v * 4 + j);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const double d[4] = {(double)ar[j].x, (double)ar[j].y, (double)ar[j].z, (double)ar[j].w};
                const double s4 = xadd(xadd(d[0], d[1]), xadd(d[2], d[3]));
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const uint32_t w = ((const uint32_t*)&m[g])[j];
                    if (w == 0) continue;
                    if (w == 0x01010101u) { acc[g] = xadd(acc[g], s4); cnt[g] += 4; continue; }
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (w & (0xffu << (8 * e))) { acc[g] = xadd(acc[g], d[e]); ++cnt[g]; }
                }
            }
        }
        done = nv << 4;
    }
    for (long long i = done + tid; i < n; i += nthreads) {
        const double d = (double)area[i];
#pragma unroll
        for (int g = 0; g < G; ++g)
            if (a.mask[g][i] != 0) { acc[g] = xadd(acc[g], d); ++cnt[g]; }
    }
    area_commit<G, BLOCK / 32>(a, acc, cnt);
}

// Bulk-copy form (default for aligned planes): the G mask planes -- G of the 4 + G B/texel -- travel
// through a shared-memory ring filled by one producer lane with G cp.async.bulk copies per stage
// (bulk.cuh), so the mask stream runs ahead of the consumers whatever they are waiting for; the area
// vector of a 16-texel step is still fetched only where some mask of the group has a texel (register
// loads, the one dependent round trip left, overlapped across 8 consumer warps x the resident
// blocks).  The register form above holds the next step's masks in registers (128 B per thread at 128
// registers, two blocks per SM): ncu r1 24 % warps active, long_scoreboard on top, 0.78 of the DRAM peak.
#ifndef ML_AREA_STAGES
#define ML_AREA_STAGES 3                               // for groups of 8 masks (28 KB stages); smaller groups get deeper rings
#endif
#ifndef ML_AREA_CW
#define ML_AREA_CW 7                                   // + the producer warp = 8 warps: 128 registers per thread at two blocks per SM
#endif
template <int G> struct AreaStages { static constexpr int N = G >= 8 ? ML_AREA_STAGES : (G >= 4 ? 4 : 6); };
constexpr int AB_CW = ML_AREA_CW;                      // consumer warps
constexpr int AB_THREADS = 32 * (AB_CW + 1);
constexpr int AB_TEXELS = 16 * 32 * AB_CW;             // texels (= bytes per mask plane) per chunk

template <int G>
__global__ void __launch_bounds__(AB_THREADS, 2)
area_bulk_kernel(const float* __restrict__ area, AreaArgs a, long long n) {
    constexpr int AB_STAGES = AreaStages<G>::N;
    typedef BulkRing<AB_STAGES, G * AB_TEXELS> Ring;
    extern __shared__ __align__(128) uint8_t ab_smem[];
    Ring& ring = *reinterpret_cast<Ring*>(ab_smem);
    double acc[G];
    unsigned cnt[G];
#pragma unroll
    for (int g = 0; g < G; ++g) { acc[g] = 0.0; cnt[g] = 0; }
    const long long nv = n >> 4;                            // whole 16-texel vectors
    const long long vbytes = nv << 4;
    const long long nchunks = (vbytes + AB_TEXELS - 1) / AB_TEXELS;
    if (threadIdx.x == 0) ring.init(AB_CW);
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    RingPos<AB_STAGES> pos;
    if (warp == AB_CW) {
        if ((threadIdx.x & 31) == 0) {
            const uint64_t policy = l2_policy_evict_first();
            for (long long c = blockIdx.x; c < nchunks; c += gridDim.x, pos.next()) {
                const long long base = c * AB_TEXELS;
                const unsigned bytes = (unsigned)(vbytes - base < AB_TEXELS ? vbytes - base : AB_TEXELS);
                ring.begin_fill(pos, bytes * G);
#pragma unroll
                for (int g = 0; g < G; ++g) ring.fill(pos, g * AB_TEXELS, a.mask[g] + base, bytes, policy);
            }
        }
    } else {
        // Two-deep software pipeline per thread: the area loads of chunk c are in flight while the masks of chunk
        // c + 1 are looked at and ITS area loads are issued; only then is chunk c accumulated -- from the masks still
        // sitting in its ring stage, which is released afterwards (so a block holds two stages while a third fills:
        // AB_STAGES >= 3).  One vector per thread and chunk with an immediate accumulate left a dependent DRAM round
        // trip exposed per step (ncu r2: long_scoreboard 10.8 per issue at 24 % issue-active).
        const unsigned off = (unsigned)threadIdx.x << 4;
        float4 ap[4];                       // area vector of the previous chunk, in flight / waiting
        RingPos<AB_STAGES> held;            // the previous chunk's stage
        unsigned held_bytes = 0;
        bool have = false, holding = false;
        auto accumulate = [&](const uint8_t* b, unsigned bytes, const float4 (&ar)[4]) {
            uint4 m[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                m[g] = make_uint4(0u, 0u, 0u, 0u);
                if (off < bytes) m[g] = *(const uint4*)(b + g * AB_TEXELS + off);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const double d[4] = {(double)ar[j].x, (double)ar[j].y, (double)ar[j].z, (double)ar[j].w};
                const double s4 = xadd(xadd(d[0], d[1]), xadd(d[2], d[3]));
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const uint32_t w = ((const uint32_t*)&m[g])[j];
                    if (w == 0) continue;
                    if (w == 0x01010101u) { acc[g] = xadd(acc[g], s4); cnt[g] += 4; continue; }
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (w & (0xffu << (8 * e))) { acc[g] = xadd(acc[g], d[e]); ++cnt[g]; }
                }
            }
        };
        for (long long c = blockIdx.x; c < nchunks; c += gridDim.x, pos.next()) {
            const long long base = c * AB_TEXELS;
            const unsigned bytes = (unsigned)(vbytes - base < AB_TEXELS ? vbytes - base : AB_TEXELS);
            const uint8_t* b = ring.acquire(pos);
            uint32_t anyset = 0;
            if (off < bytes) {
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const uint4 m = *(const uint4*)(b + g * AB_TEXELS + off);
                    anyset |= m.x | m.y | m.z | m.w;
                }
            }
            float4 ar[4];
            if (anyset) {
                const float4* ap4 = (const float4*)(area + base + off);
#pragma unroll
                for (int j = 0; j < 4; ++j) ar[j] = ld_stream(ap4 + j);
            }
            if (holding) {
                if (have) accumulate(ring.buf[held.stage], held_bytes, ap);
                ring.release(held);
            }
            held = pos; held_bytes = bytes; holding = true;
            have = anyset != 0;
            if (have) {
#pragma unroll
                for (int j = 0; j < 4; ++j) ap[j] = ar[j];
            }
        }
        if (holding) {
            if (have) accumulate(ring.buf[held.stage], held_bytes, ap);
            ring.release(held);
        }
        if (blockIdx.x == 0) {
            for (long long i = vbytes + threadIdx.x; i < n; i += 32 * AB_CW) {     // < 16 texels of tail
                const double d = (double)area[i];
#pragma unroll
                for (int g = 0; g < G; ++g)
                    if (a.mask[g][i] != 0) { acc[g] = xadd(acc[g], d); ++cnt[g]; }
            }
        }
    }
    // block reduction over all AB_THREADS threads (the producer warp contributes zeros)
    area_commit<G, AB_CW + 1>(a, acc, cnt);
}

inline bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

template <int G>
int launch_area_bulk(const float* area, const AreaArgs& a, long long n, cudaStream_t st) {
    typedef BulkRing<AreaStages<G>::N, G * AB_TEXELS> Ring;
    static int per_sm = 0;
    const void* fn = (const void*)area_bulk_kernel<G>;
    if (!per_sm) {
        ML_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Ring)));
        int nb = 0;
        ML_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, AB_THREADS, sizeof(Ring)));
        per_sm = nb > 0 ? nb : 1;
    }
    const long long nchunks = (((n >> 4) << 4) + AB_TEXELS - 1) / AB_TEXELS;
    long long blocks = (long long)ml_sm_count() * per_sm;
    if (blocks > nchunks) blocks = nchunks;
    if (blocks < 1) blocks = 1;
    area_bulk_kernel<G><<<(unsigned)blocks, AB_THREADS, sizeof(Ring), st>>>(area, a, n);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

template <int G>
int launch_area(const float* area, const AreaArgs& a, long long n, cudaStream_t st) {
    bool vec = aligned16(area);
    for (int g = 0; g < G; ++g) vec = vec && aligned16(a.mask[g]);
    static const bool reg_form = getenv("ML_AREA_REGISTER_STREAM") != nullptr;       // the round-1 kernel, kept for comparison
    if (vec && !reg_form && n >= 4 * AB_TEXELS) return launch_area_bulk<G>(area, a, n, st);
    const long long items = vec ? ((n + 15) >> 4) : n;
    long long blocks = (items + BLOCK - 1) / BLOCK;
    const long long cap = (long long)ml_sm_count() * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    if (vec) area_kernel<G, true><<<(unsigned)blocks, BLOCK, 0, st>>>(area, a, n);
    else area_kernel<G, false><<<(unsigned)blocks, BLOCK, 0, st>>>(area, a, n);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

// ---------------------------------------------------------------------------------------------
// area per label of a uint8 plane: per-block shared-memory bins, run-length aggregation per
// thread (labels are spatially coherent), one global atomic per non-empty bin per block.
__global__ void __launch_bounds__(BLOCK)
label_area_kernel(const float* __restrict__ area, const uint8_t* __restrict__ data,
                  const uint8_t* __restrict__ mask, long long n, double* sums, unsigned long long* counts) {
    __shared__ double s_sum[256];
    __shared__ unsigned long long s_cnt[256];
    for (int v = threadIdx.x; v < 256; v += BLOCK) { s_sum[v] = 0.0; s_cnt[v] = 0; }
    __syncthreads();
    const long long nthreads = (long long)gridDim.x * BLOCK;
    const long long per = 16;
    const long long nchunks = (n + per - 1) / per;
    for (long long c = (long long)blockIdx.x * BLOCK + threadIdx.x; c < nchunks; c += nthreads) {
        const long long b = c * per, e = (b + per < n) ? b + per : n;
        int run = -1; double rs = 0.0; unsigned long long rc = 0;
        for (long long i = b; i < e; ++i) {
            if (mask[i] == 0) continue;
            const int v = data[i];
            if (v != run) {
                if (rc) { atomicAdd(&s_sum[run], rs); atomicAdd(&s_cnt[run], rc); }
                run = v; rs = 0.0; rc = 0;
            }
            rs = xadd(rs, (double)area[i]); ++rc;
        }
        if (rc) { atomicAdd(&s_sum[run], rs); atomicAdd(&s_cnt[run], rc); }
    }
    __syncthreads();
    for (int v = threadIdx.x; v < 256; v += BLOCK)
        if (s_cnt[v]) { atomicAdd(sums + v, s_sum[v]); atomicAdd(counts + v, s_cnt[v]); }
}

// ---------------------------------------------------------------------------------------------
template <typename T> ML_DEV double widen(T v) { return (double)v; }
struct HalfBits { uint16_t b; };
template <> ML_DEV double widen<HalfBits>(HalfBits v) {
    // IEEE binary16 -> float64 without <cuda_fp16.h> conversions (exact)
    const uint32_t sign = (uint32_t)(v.b >> 15) << 31, ex = (v.b >> 10) & 31u, man = v.b & 1023u;
    uint32_t bits;
    if (ex == 0) {
        if (man == 0) bits = sign;
        else {
            int sh = 0; uint32_t m = man;
            while (!(m & 1024u)) { m <<= 1; ++sh; }
            bits = sign | ((uint32_t)(113 - sh) << 23) | ((m & 1023u) << 13);
        }
    } else if (ex == 31) bits = sign | 0x7f800000u | (man << 13);
    else bits = sign | ((ex + 112u) << 23) | (man << 13);
    return (double)__uint_as_float(bits);
}

ML_DEV void atomic_min_double(double* p, double v) {
    unsigned long long* a = (unsigned long long*)p;
    unsigned long long old = *a;
    while (v < __longlong_as_double((long long)old)) {
        const unsigned long long assumed = old;
        old = atomicCAS(a, assumed, (unsigned long long)__double_as_longlong(v));
        if (old == assumed) break;
    }
}
ML_DEV void atomic_max_double(double* p, double v) {
    unsigned long long* a = (unsigned long long*)p;
    unsigned long long old = *a;
    while (v > __longlong_as_double((long long)old)) {
        const unsigned long long assumed = old;
        old = atomicCAS(a, assumed, (unsigned long long)__double_as_longlong(v));
        if (old == assumed) break;
    }
}

// 16 texels per thread and step: one 128-bit mask load + sizeof(T) 128-bit attribute loads, two steps
// in flight; VEC = false (unaligned planes) and the tail take the scalar loop.  The float64 sum is
// accumulated per thread, then warp shuffle -> one atomic per block (order-free within 1e-10, the
// oracle comparison tolerance; count / min / max are exact).
template <typename T, bool VEC>
__global__ void __launch_bounds__(BLOCK)
stats_kernel(const T* __restrict__ attr, const uint8_t* __restrict__ mask, long long n, double* out) {
    __shared__ double s_mn[BLOCK / 32], s_mx[BLOCK / 32];
    double sum = 0.0, mn = INFINITY, mx = -INFINITY;
    long long cnt = 0;
    const long long tid = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * BLOCK;
    long long done = 0;
    if (VEC) {
        constexpr int W = (int)sizeof(T);                    // 128-bit words per 16 attributes
        struct __align__(16) Vec { T v[16]; };
        const long long nv = n >> 4;
        for (long long v0 = tid; v0 < nv; v0 += 2 * nthreads) {
            uint4 m[2];
            Vec a[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const long long v = v0 + u * nthreads;
                m[u] = make_uint4(0, 0, 0, 0);
                if (v < nv) {
                    m[u] = ld_stream((const uint4*)mask + v);
#pragma unroll
                    for (int k = 0; k < W; ++k) ((uint4*)&a[u])[k] = ld_stream((const uint4*)attr + v * W + k);
                }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const uint32_t mw[4] = {m[u].x, m[u].y, m[u].z, m[u].w};
                if ((mw[0] | mw[1] | mw[2] | mw[3]) == 0) continue;
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    if (((mw[e >> 2] >> (8 * (e & 3))) & 0xffu) == 0) continue;
                    const double x = widen(a[u].v[e]);
                    sum = xadd(sum, x); ++cnt;
                    if (x < mn) mn = x;
                    if (x > mx) mx = x;
                }
            }
        }
        done = nv << 4;
    }
    for (long long i = done + tid; i < n; i += nthreads) {
        if (mask[i] == 0) continue;
        const double v = widen(attr[i]);
        sum = xadd(sum, v); ++cnt;
        if (v < mn) mn = v;
        if (v > mx) mx = v;
    }
    // count is accumulated as a double: exact below 2^53 texels
    block_sum_atomic((double)cnt, out);
    block_sum_atomic(sum, out + 1);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) { s_mn[wid] = mn; s_mx[wid] = mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < BLOCK / 32; ++w) { mn = fmin(mn, s_mn[w]); mx = fmax(mx, s_mx[w]); }
        atomic_min_double(out + 2, mn);
        atomic_max_double(out + 3, mx);
    }
}

template <typename T>
int launch_stats(const void* attr, const uint8_t* mask, long long n, double* out, cudaStream_t st) {
    const bool vec = ((((uintptr_t)attr) | ((uintptr_t)mask)) & 15) == 0;
    long long blocks = ((vec ? (n + 31) / 32 : n) + BLOCK - 1) / BLOCK;
    const long long cap = (long long)ml_sm_count() * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    if (vec) stats_kernel<T, true><<<(unsigned)blocks, BLOCK, 0, st>>>((const T*)attr, mask, n, out);
    else stats_kernel<T, false><<<(unsigned)blocks, BLOCK, 0, st>>>((const T*)attr, mask, n, out);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

}  // namespace

extern "C" {

static int layer_area_groups(const float* area, const uint8_t* const* masks, int64_t L, int64_t n, double* sums,
                             uint64_t* counts, void* const* peer_rows, int npeers, cudaStream_t st) {
    for (int64_t l0 = 0; l0 < L; ) {
        const int64_t left = L - l0;
        const int g = left >= 8 ? 8 : left >= 4 ? 4 : left >= 2 ? 2 : 1;
        AreaArgs a;
        for (int k = 0; k < MAX_G; ++k) a.mask[k] = k < g ? masks[l0 + k] : nullptr;
        a.sums = sums ? sums + l0 : nullptr;
        a.counts = counts ? (unsigned long long*)counts + l0 : nullptr;
        a.npeers = npeers;
        for (int p = 0; p < MAX_PEERS; ++p) {
            a.peer_sums[p] = p < npeers ? (double*)peer_rows[p] + l0 : nullptr;
            a.peer_counts[p] = p < npeers ? (unsigned long long*)peer_rows[p] + L + l0 : nullptr;
        }
        int rc;
        switch (g) {
        case 8: rc = launch_area<8>(area, a, n, st); break;
        case 4: rc = launch_area<4>(area, a, n, st); break;
        case 2: rc = launch_area<2>(area, a, n, st); break;
        default: rc = launch_area<1>(area, a, n, st); break;
        }
        if (rc != ML_OK) return rc;
        l0 += g;
    }
    return ML_OK;
}

int ml_layer_area(const float* area, const uint8_t* const* masks, int64_t L, int64_t n,
                  double* sums, uint64_t* counts, void* stream) {
    if (L < 0 || L > 64) return ml_fail(ML_ERR_ARG, "layer count must be 0..64");
    if (n <= 0) return ML_OK;
    return layer_area_groups(area, masks, L, n, sums, counts, nullptr, 0, (cudaStream_t)stream);
}

// Signal + wait of the fused cross-rank reduction: ONE thread tells every rank (system-scope atomic on its row's
// arrival slot) that this rank's contributions are complete, then waits until all `target` ranks have told THIS rank.
// Bounded: after ~10 s without progress it raises *status instead of hanging the GPU.
__global__ void peer_arrive_wait_kernel(unsigned long long* const* arrive, int npeers, const volatile unsigned long long* own,
                                        unsigned long long target, unsigned int* status) {
    __threadfence_system();
    for (int p = 0; p < npeers; ++p) atomicAdd_system(arrive[p], 1ull);
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (*own < target) {
        __nanosleep(200);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > 10000000000ull) { if (status) atomicExch(status, 1u); break; }
    }
    __threadfence_system();
}

int ml_layer_area_peers(const float* area, const uint8_t* const* masks, int64_t L, int64_t n,
                        void* const* peer_rows, int npeers, int self, void* arrive_table, uint32_t* status,
                        void* recycle_row, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (L < 0 || L > 64) return ml_fail(ML_ERR_ARG, "layer count must be 0..64");
    if (npeers < 1 || npeers > MAX_PEERS || self < 0 || self >= npeers || peer_rows == nullptr || arrive_table == nullptr)
        return ml_fail(ML_ERR_ARG, "ml_layer_area_peers: 1..16 peers, self among them, row pointers and the arrival table");
    if (n > 0) {
        const int rc = layer_area_groups(area, masks, L, n, nullptr, nullptr, peer_rows, npeers, st);
        if (rc != ML_OK) return rc;
    }
    // arrive_table: device array of npeers pointers = the arrival slot (u64 at index 2L) of every rank's row
    const volatile unsigned long long* own = (const volatile unsigned long long*)peer_rows[self] + 2 * L;
    peer_arrive_wait_kernel<<<1, 1, 0, st>>>((unsigned long long* const*)arrive_table, npeers, own, (unsigned long long)npeers, status);
    ML_CUDA(cudaGetLastError());
    if (recycle_row) ML_CUDA(cudaMemsetAsync(recycle_row, 0, (size_t)(2 * L + 2) * sizeof(unsigned long long), st));
    return ML_OK;
}

// Peer memory for the fused reduction: plain cudaMalloc regions (IPC handles need allocation bases, which torch's
// caching allocator does not hand out), exported / opened as 64-byte cudaIpcMemHandle_t blobs.
int ml_peer_alloc(void** ptr, size_t bytes) {
    if (!ptr) return ml_fail(ML_ERR_ARG, "ml_peer_alloc: null");
    ML_CUDA(cudaMalloc(ptr, bytes ? bytes : 1));
    ML_CUDA(cudaMemset(*ptr, 0, bytes ? bytes : 1));
    return ML_OK;
}
int ml_peer_free(void* ptr) { if (ptr) ML_CUDA(cudaFree(ptr)); return ML_OK; }
int ml_peer_export(const void* ptr, void* handle64) {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handles are 64 bytes");
    cudaIpcMemHandle_t h;
    ML_CUDA(cudaIpcGetMemHandle(&h, (void*)ptr));
    memcpy(handle64, &h, 64);
    return ML_OK;
}
int ml_peer_open(const void* handle64, void** ptr) {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    ML_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return ML_OK;
}
int ml_peer_close(void* ptr) { if (ptr) ML_CUDA(cudaIpcCloseMemHandle(ptr)); return ML_OK; }
// 1 iff the current device can run native atomics on memory of `peer_device` (same device: always)
int ml_peer_atomics_supported(int peer_device) {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (dev == peer_device) return 1;
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, dev, peer_device) != cudaSuccess || !can) return 0;
    if (cudaDeviceGetP2PAttribute(&v, cudaDevP2PAttrNativeAtomicSupported, dev, peer_device) != cudaSuccess) return 0;
    return v ? 1 : 0;
}

int ml_label_area(const float* area, const uint8_t* data, const uint8_t* mask, int64_t n,
                  double* sums, uint64_t* counts, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) return ML_OK;
    long long blocks = ((n + 15) / 16 + BLOCK - 1) / BLOCK;
    const long long cap = (long long)ml_sm_count() * 8;
    if (blocks > cap) blocks = cap;
    label_area_kernel<<<(unsigned)blocks, BLOCK, 0, st>>>(area, data, mask, n, sums, (unsigned long long*)counts);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int ml_layer_stats(const void* attr, int attr_kind, const uint8_t* mask, int64_t n,
                   double* out, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) return ML_OK;
    switch (attr_kind) {
    case ML_U8:  return launch_stats<uint8_t>(attr, mask, n, out, st);
    case ML_I8:  return launch_stats<int8_t>(attr, mask, n, out, st);
    case ML_I16: return launch_stats<int16_t>(attr, mask, n, out, st);
    case ML_I32: return launch_stats<int32_t>(attr, mask, n, out, st);
    case ML_U32: return launch_stats<uint32_t>(attr, mask, n, out, st);
    case ML_F16: return launch_stats<HalfBits>(attr, mask, n, out, st);
    case ML_FLOAT32: return launch_stats<float>(attr, mask, n, out, st);
    }
    return ml_fail(ML_ERR_ARG, "unknown attribute kind");
}

}  // extern "C"
