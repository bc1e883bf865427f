// Selection brushes (north star (2)): sphere brush over the position map and attribute-threshold
// selection.  No reference code exists for them; the frozen definitions are
// oracle/kn_port.c ext_select_sphere / ext_select_sphere_batch / ext_select_threshold, and the
// write rule is the reference's (KN:198-202: count 0 -> 1 edits, data = value, mask = 1,
// edited = 1).
//
// Both are pure streams: 12 B/texel (three float32 position planes) resp. attr + valid bytes,
// read once with 128-bit no-allocate loads; writes happen only for hits.  Every thread keeps
// UNROLL independent 16-byte loads per plane in flight.
#include <cuda_fp16.h>
#include "common.cuh"
#include "meshlayers_b200.h"
#include "internal.h"

namespace {

constexpr int BLOCK = 256;
constexpr int UNROLL = 4;

ML_DEV void hit_write(void* data, int esize, uint32_t value, uint8_t* mask, uint8_t* edited,
                      long long i, long long& cnt) {
    if (edited[i] == 0) ++cnt;
    store_value(data, esize, i, value);
    mask[i] = 1;
    edited[i] = 1;
}

ML_DEV bool sphere_hit(float px, float py, float pz, double cx, double cy, double cz, double r2) {
    const double dx = xsub((double)px, cx), dy = xsub((double)py, cy), dz = xsub((double)pz, cz);
    const double d2 = xadd(xadd(xmul(dx, dx), xmul(dy, dy)), xmul(dz, dz));
    return d2 <= r2;
}

ML_DEV bool sphere_hit_d(double px, double py, double pz, double cx, double cy, double cz, double r2) {
    const double dx = xsub(px, cx), dy = xsub(py, cy), dz = xsub(pz, cz);
    const double d2 = xadd(xadd(xmul(dx, dx), xmul(dy, dy)), xmul(dz, dz));
    return d2 <= r2;
}

// VEC = 4: 128-bit loads (planes 16-byte aligned); VEC = 1: scalar fallback for odd alignments.
template <int VEC>
__global__ void __launch_bounds__(BLOCK)
sphere_kernel(const float* __restrict__ px, const float* __restrict__ py, const float* __restrict__ pz,
              long long n, double cx, double cy, double cz, double r2,
              void* __restrict__ data, int esize, uint32_t value,
              uint8_t* __restrict__ mask, uint8_t* __restrict__ edited, unsigned long long* counter) {
    long long cnt = 0;
    const long long tid = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * BLOCK;
    if (VEC == 4) {
        const long long nq = n >> 2;
        const float4* qx = (const float4*)px; const float4* qy = (const float4*)py; const float4* qz = (const float4*)pz;
        for (long long q0 = tid; q0 < nq; q0 += nthreads * UNROLL) {
            float4 vx[UNROLL], vy[UNROLL], vz[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const long long q = q0 + u * nthreads;
                if (q < nq) { vx[u] = ld_stream(qx + q); vy[u] = ld_stream(qy + q); vz[u] = ld_stream(qz + q); }
            }
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const long long q = q0 + u * nthreads;
                if (q >= nq) break;
                const long long i = q << 2;
                if (sphere_hit(vx[u].x, vy[u].x, vz[u].x, cx, cy, cz, r2)) hit_write(data, esize, value, mask, edited, i, cnt);
                if (sphere_hit(vx[u].y, vy[u].y, vz[u].y, cx, cy, cz, r2)) hit_write(data, esize, value, mask, edited, i + 1, cnt);
                if (sphere_hit(vx[u].z, vy[u].z, vz[u].z, cx, cy, cz, r2)) hit_write(data, esize, value, mask, edited, i + 2, cnt);
                if (sphere_hit(vx[u].w, vy[u].w, vz[u].w, cx, cy, cz, r2)) hit_write(data, esize, value, mask, edited, i + 3, cnt);
            }
        }
        for (long long i = (nq << 2) + tid; i < n; i += nthreads)
            if (sphere_hit(px[i], py[i], pz[i], cx, cy, cz, r2)) hit_write(data, esize, value, mask, edited, i, cnt);
    } else {
        for (long long i = tid; i < n; i += nthreads)
            if (sphere_hit(px[i], py[i], pz[i], cx, cy, cz, r2)) hit_write(data, esize, value, mask, edited, i, cnt);
    }
    block_count_add(cnt, counter);
}

// ---------------------------------------------------------------------------------------------
// K strokes in one pass.  Each block owns TILE consecutive texels per iteration:
//   1. streams the tile's positions into registers and reduces their bounding box,
//   2. culls the stroke list against the box (conservative float64 sphere/box test) into an
//      ORDER-PRESERVING list in shared memory,
//   3. every texel tests only the surviving strokes, in stroke order, so the result equals K
//      successive single-stroke passes (later strokes overwrite earlier ones).
constexpr int TILE_Q = BLOCK;             // quads per tile -> TILE = 1024 texels
constexpr int MAX_LIST = 1024;            // surviving strokes kept per tile pass

struct BatchArgs {
    const float *px, *py, *pz;
    long long n;
    const double* strokes; const int* layer_of; const uint32_t* value_bits; long long K;
    void* const* data; uint8_t* const* mask; uint8_t* const* edited; long long L;
    int esize; unsigned long long* counts;
};

ML_DEV float warp_min(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
ML_DEV float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__global__ void __launch_bounds__(BLOCK)
sphere_batch_kernel(BatchArgs a) {
    __shared__ float s_lo[3][BLOCK / 32], s_hi[3][BLOCK / 32];
    __shared__ double s_box[6];
    __shared__ int s_list[MAX_LIST];
    __shared__ double s_sph[MAX_LIST][4];
    __shared__ int s_wcount[BLOCK / 32];
    __shared__ int s_nlist;
    __shared__ unsigned long long s_counts[64];
    const bool smem_counts = a.L <= 64;
    if (threadIdx.x < 64) s_counts[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long nq = a.n >> 2;                       // host guarantees n % 4 == 0 handled by tail call
    const long long ntiles = (nq + TILE_Q - 1) / TILE_Q;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long q = tile * TILE_Q + threadIdx.x;
        const bool live = q < nq;
        float4 vx, vy, vz;
        const float inf = __int_as_float(0x7f800000);
        float lo[3] = {inf, inf, inf}, hi[3] = {-inf, -inf, -inf};
        if (live) {
            vx = ld_stream((const float4*)a.px + q);
            vy = ld_stream((const float4*)a.py + q);
            vz = ld_stream((const float4*)a.pz + q);
            // fminf / fmaxf ignore NaN (uncovered texels)
            lo[0] = fminf(fminf(vx.x, vx.y), fminf(vx.z, vx.w)); hi[0] = fmaxf(fmaxf(vx.x, vx.y), fmaxf(vx.z, vx.w));
            lo[1] = fminf(fminf(vy.x, vy.y), fminf(vy.z, vy.w)); hi[1] = fmaxf(fmaxf(vy.x, vy.y), fmaxf(vy.z, vy.w));
            lo[2] = fminf(fminf(vz.x, vz.y), fminf(vz.z, vz.w)); hi[2] = fmaxf(fmaxf(vz.x, vz.y), fmaxf(vz.z, vz.w));
            // a NaN-only component leaves lo = NaN? no: fminf(NaN, NaN) = NaN -> normalise
#pragma unroll
            for (int c = 0; c < 3; ++c) { if (!(lo[c] == lo[c])) lo[c] = inf; if (!(hi[c] == hi[c])) hi[c] = -inf; }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float l = warp_min(lo[c]), h = warp_max(hi[c]);
            if (lane == 0) { s_lo[c][wid] = l; s_hi[c][wid] = h; }
        }
        __syncthreads();
        if (threadIdx.x < 3) {
            float l = s_lo[threadIdx.x][0], h = s_hi[threadIdx.x][0];
            for (int w = 1; w < BLOCK / 32; ++w) { l = fminf(l, s_lo[threadIdx.x][w]); h = fmaxf(h, s_hi[threadIdx.x][w]); }
            s_box[threadIdx.x] = (double)l; s_box[3 + threadIdx.x] = (double)h;
        }
        __syncthreads();
        const double bl0 = s_box[0], bl1 = s_box[1], bl2 = s_box[2], bh0 = s_box[3], bh1 = s_box[4], bh2 = s_box[5];
        const bool empty_box = !(bl0 <= bh0);             // tile holds no covered texel
        // stroke passes: cull MAX_LIST-sized, order-preserving batches
        for (long long k0 = 0; k0 < a.K && !empty_box; ) {
            if (threadIdx.x == 0) s_nlist = 0;
            __syncthreads();
            long long k = k0;
            // rounds of BLOCK strokes until the list is (nearly) full or strokes are exhausted
            while (k < a.K) {
                const long long kk = k + threadIdx.x;
                bool keep = false;
                double sx = 0, sy = 0, sz = 0, sr = 0;
                if (kk < a.K) {
                    sx = a.strokes[4 * kk]; sy = a.strokes[4 * kk + 1]; sz = a.strokes[4 * kk + 2]; sr = a.strokes[4 * kk + 3];
                    // distance from the centre to the box, per axis max(lo-c, 0, c-hi)
                    const double ddx = fmax(fmax(xsub(bl0, sx), xsub(sx, bh0)), 0.0);
                    const double ddy = fmax(fmax(xsub(bl1, sy), xsub(sy, bh1)), 0.0);
                    const double ddz = fmax(fmax(xsub(bl2, sz), xsub(sz, bh2)), 0.0);
                    const double dmin2 = xadd(xadd(xmul(ddx, ddx), xmul(ddy, ddy)), xmul(ddz, ddz));
                    // every texel p of the tile has fl(d2(p)) >= dmin2*(1-8u); keep unless the box
                    // is provably outside: dmin2 > r2*(1+1e-12)
                    keep = !(dmin2 > xmul(xmul(sr, sr), 1.000000000001));
                }
                const unsigned bal = __ballot_sync(0xffffffffu, keep);
                if (lane == 0) s_wcount[wid] = __popc(bal);
                __syncthreads();
                int base = s_nlist, before = 0, total = 0;
                for (int w = 0; w < BLOCK / 32; ++w) { if (w < wid) before += s_wcount[w]; total += s_wcount[w]; }
                const bool fits = base + total <= MAX_LIST;
                if (fits && keep) {
                    const int slot = base + before + __popc(bal & ((1u << lane) - 1u));
                    s_list[slot] = (int)kk;
                    s_sph[slot][0] = sx; s_sph[slot][1] = sy; s_sph[slot][2] = sz; s_sph[slot][3] = xmul(sr, sr);
                }
                __syncthreads();
                if (!fits) break;                         // process what we have, resume at k
                if (threadIdx.x == 0) s_nlist = base + total;
                k += BLOCK;
                __syncthreads();
            }
            k0 = (k < a.K) ? k : a.K;
            const int nl = s_nlist;
            if (live && nl > 0) {
                const double fx[4] = {(double)vx.x, (double)vx.y, (double)vx.z, (double)vx.w};
                const double fy[4] = {(double)vy.x, (double)vy.y, (double)vy.z, (double)vy.w};
                const double fz[4] = {(double)vz.x, (double)vz.y, (double)vz.z, (double)vz.w};
                for (int j = 0; j < nl; ++j) {
                    const double sx = s_sph[j][0], sy = s_sph[j][1], sz = s_sph[j][2], r2 = s_sph[j][3];
                    unsigned hits = 0;
#pragma unroll
                    for (int e = 0; e < 4; ++e) if (sphere_hit_d(fx[e], fy[e], fz[e], sx, sy, sz, r2)) hits |= 1u << e;
                    if (hits) {
                        const int kk = s_list[j];
                        const int layer = a.layer_of[kk];
                        const uint32_t value = a.value_bits[kk];
                        void* d = a.data[layer]; uint8_t* m = a.mask[layer]; uint8_t* ed = a.edited[layer];
                        long long c = 0;
#pragma unroll
                        for (int e = 0; e < 4; ++e) if (hits & (1u << e)) hit_write(d, a.esize, value, m, ed, (q << 2) + e, c);
                        if (c) atomicAdd(smem_counts ? &s_counts[layer] : a.counts + layer, (unsigned long long)c);
                    }
                }
            }
            __syncthreads();
        }
        __syncthreads();
    }
    if (smem_counts && threadIdx.x < a.L && s_counts[threadIdx.x]) atomicAdd(a.counts + threadIdx.x, s_counts[threadIdx.x]);
}

// ---------------------------------------------------------------------------------------------
template <int KIND> struct AttrT;
template <> struct AttrT<ML_U8>  { typedef uint8_t T;  static ML_DEV double get(T v) { return (double)v; } };
template <> struct AttrT<ML_I8>  { typedef int8_t T;   static ML_DEV double get(T v) { return (double)v; } };
template <> struct AttrT<ML_I16> { typedef int16_t T;  static ML_DEV double get(T v) { return (double)v; } };
template <> struct AttrT<ML_I32> { typedef int32_t T;  static ML_DEV double get(T v) { return (double)v; } };
template <> struct AttrT<ML_U32> { typedef uint32_t T; static ML_DEV double get(T v) { return (double)v; } };
template <> struct AttrT<ML_F16> { typedef uint16_t T; static ML_DEV double get(T v) { return (double)__half2float(__ushort_as_half(v)); } };
template <> struct AttrT<ML_FLOAT32> { typedef float T; static ML_DEV double get(T v) { return (double)v; } };

// 4 texels per step: one (4*sizeof(T))-byte attribute load + one 4-byte valid load.
template <int KIND, bool VECTOR>
__global__ void __launch_bounds__(BLOCK)
threshold_kernel(const void* __restrict__ attr_, const uint8_t* __restrict__ valid, long long n,
                 double lo, double hi, void* __restrict__ data, int esize, uint32_t value,
                 uint8_t* __restrict__ mask, uint8_t* __restrict__ edited, unsigned long long* counter) {
    typedef typename AttrT<KIND>::T T;
    const T* attr = (const T*)attr_;
    long long cnt = 0;
    const long long tid = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * BLOCK;
    long long done = 0;
    if (VECTOR) {
        struct __align__(sizeof(T) * 4) Quad { T v[4]; };
        const long long nq = n >> 2;
        for (long long q0 = tid; q0 < nq; q0 += nthreads * UNROLL) {
            Quad a[UNROLL]; uint32_t vm[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const long long q = q0 + u * nthreads;
                if (q < nq) {
                    a[u] = ((const Quad*)attr)[q];
                    vm[u] = valid ? ld_stream((const uint32_t*)valid + q) : 0x01010101u;
                }
            }
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const long long q = q0 + u * nthreads;
                if (q >= nq) break;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (((vm[u] >> (8 * e)) & 0xffu) == 0) continue;
                    const double v = AttrT<KIND>::get(a[u].v[e]);
                    if (lo <= v && v <= hi) hit_write(data, esize, value, mask, edited, (q << 2) + e, cnt);
                }
            }
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

inline unsigned stream_grid(long long items_per_thread_iter, long long n_items) {
    long long blocks = (n_items + (long long)BLOCK * items_per_thread_iter - 1) / ((long long)BLOCK * items_per_thread_iter);
    const long long cap = (long long)ml_sm_count() * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (unsigned)blocks;
}

inline bool aligned(const void* p, size_t a) { return ((uintptr_t)p % a) == 0; }

template <int KIND>
int launch_threshold(const void* attr, const uint8_t* valid, long long n, double lo, double hi,
                     void* data, int esize, uint32_t value, uint8_t* mask, uint8_t* edited,
                     unsigned long long* counter, cudaStream_t st) {
    typedef typename AttrT<KIND>::T T;
    const bool vec = aligned(attr, sizeof(T) * 4) && (!valid || aligned(valid, 4));
    const unsigned grid = stream_grid(4 * UNROLL, n);
    if (vec) threshold_kernel<KIND, true><<<grid, BLOCK, 0, st>>>(attr, valid, n, lo, hi, data, esize, value, mask, edited, counter);
    else threshold_kernel<KIND, false><<<grid, BLOCK, 0, st>>>(attr, valid, n, lo, hi, data, esize, value, mask, edited, counter);
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
    const bool vec = aligned(px, 16) && aligned(py, 16) && aligned(pz, 16);
    const unsigned grid = stream_grid(4 * UNROLL, n);
    if (vec) sphere_kernel<4><<<grid, BLOCK, 0, st>>>(px, py, pz, n, cx, cy, cz, r2, data, esize, value_bits, mask, edited, (unsigned long long*)count);
    else sphere_kernel<1><<<grid, BLOCK, 0, st>>>(px, py, pz, n, cx, cy, cz, r2, data, esize, value_bits, mask, edited, (unsigned long long*)count);
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
    BatchArgs a{px, py, pz, n, strokes, layer_of, value_bits, K, data, mask, edited, L, esize,
                (unsigned long long*)counts};
    const long long ntiles = ((n >> 2) + TILE_Q - 1) / TILE_Q;
    long long blocks = ntiles;
    const long long cap = (long long)ml_sm_count() * 8;
    if (blocks > cap) blocks = cap;
    sphere_batch_kernel<<<(unsigned)blocks, BLOCK, 0, st>>>(a);
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
