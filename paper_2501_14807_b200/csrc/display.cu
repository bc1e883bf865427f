// Display resolution and mask bit-packing.
//
//   ml_resolve_display : per texel, mask ? palette(clamp((value-lower)/(upper-lower))) : transparent,
//                        written as RGBA8.  Pure stream: esize + 1 bytes read, 4 bytes written.
//   ml_pack_mask / ml_unpack_mask : byte mask plane <-> packed bits (MSB first within a byte, the
//                        numpy.packbits convention) for the L3DI layer file -- the device packs so
//                        that only n/8 bytes cross PCIe.
// The reference has no code for these; frozen definitions: oracle/kn_port.c ext_resolve_display,
// ext_pack_mask.  Colour arithmetic is unfused float64 in the order written there.
#include <cuda_fp16.h>
#include "common.cuh"
#include "meshlayers_b200.h"
#include "internal.h"

namespace {

constexpr int BLOCK = 256;
constexpr int MAX_POINTS = 64;

struct PaletteArgs {
    double pos[MAX_POINTS];
    double rgba[MAX_POINTS][4];
    int npoints;
    double lower, upper;
};

template <int KIND> struct ValT;
template <> struct ValT<ML_U8>  { typedef uint8_t T;  static ML_DEV double get(T v) { return (double)v; } };
template <> struct ValT<ML_I8>  { typedef int8_t T;   static ML_DEV double get(T v) { return (double)v; } };
template <> struct ValT<ML_I16> { typedef int16_t T;  static ML_DEV double get(T v) { return (double)v; } };
template <> struct ValT<ML_I32> { typedef int32_t T;  static ML_DEV double get(T v) { return (double)v; } };
template <> struct ValT<ML_U32> { typedef uint32_t T; static ML_DEV double get(T v) { return (double)v; } };
template <> struct ValT<ML_F16> { typedef uint16_t T; static ML_DEV double get(T v) { return (double)__half2float(__ushort_as_half(v)); } };
template <> struct ValT<ML_FLOAT32> { typedef float T; static ML_DEV double get(T v) { return (double)v; } };

// u = clamp((value - lower)/(upper - lower), 0, 1); piecewise-linear palette at u;
// channel byte = floor(c*255 + 0.5) clamped to [0, 255].  NaN values map to u = 0.
ML_DEV uint32_t colour_of(const PaletteArgs& p, double value) {
    double u = xdiv(xsub(value, p.lower), xsub(p.upper, p.lower));
    if (!(u > 0.0)) u = 0.0;
    if (u > 1.0) u = 1.0;
    int k = 0;
    while (k + 2 < p.npoints && u > p.pos[k + 1]) ++k;           // segment [pos[k], pos[k+1]] containing u
    const double t = xdiv(xsub(u, p.pos[k]), xsub(p.pos[k + 1], p.pos[k]));
    uint32_t out = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const double v = xadd(p.rgba[k][c], xmul(t, xsub(p.rgba[k + 1][c], p.rgba[k][c])));
        double b = floor(xadd(xmul(v, 255.0), 0.5));
        if (!(b > 0.0)) b = 0.0;
        if (b > 255.0) b = 255.0;
        out |= (uint32_t)b << (8 * c);                            // little-endian RGBA bytes
    }
    return out;
}

// 1-byte kinds have 256 possible values: every block first evaluates colour_of for all of them into
// shared memory (the same function, so the same bits) and the stream becomes a table lookup --
// 2 bytes read + 4 written per texel at HBM speed instead of ~80 float64 instructions per texel.
template <int KIND>
__global__ void __launch_bounds__(BLOCK)
display_kernel(const void* __restrict__ data_, const uint8_t* __restrict__ mask, long long n,
               const __grid_constant__ PaletteArgs p, uint32_t* __restrict__ rgba) {
    typedef typename ValT<KIND>::T T;
    constexpr bool LUT = sizeof(T) == 1;
    constexpr int U = 4;
    __shared__ uint32_t s_lut[LUT ? 256 : 1];
    if (LUT) {
        static_assert(BLOCK == 256, "one table entry per thread");
        s_lut[threadIdx.x] = colour_of(p, ValT<KIND>::get((T)threadIdx.x));     // T wraps 128..255 to int8 -128..-1
        __syncthreads();
    }
    const T* data = (const T*)data_;
    const long long nthreads = (long long)gridDim.x * BLOCK;
    const long long tid = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const long long nq = n >> 2;
    struct __align__(sizeof(T) * 4) Quad { T v[4]; };
    const bool vec = (((uintptr_t)data) % (sizeof(T) * 4) == 0) && (((uintptr_t)mask) % 4 == 0) && (((uintptr_t)rgba) % 16 == 0);
    long long done = 0;
    if (vec) {
        for (long long q0 = tid; q0 < nq; q0 += nthreads * U) {
            uint32_t m[U];
            Quad a[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long q = q0 + u * nthreads;
                m[u] = q < nq ? ld_stream((const uint32_t*)mask + q) : 0u;
                if (LUT && q < nq) a[u] = ld_quad((const Quad*)data + q);       // cheap enough to load unconditionally
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long q = q0 + u * nthreads;
                if (q >= nq) break;
                uint4 out = make_uint4(0, 0, 0, 0);
                if (m[u]) {
                    if (!LUT) a[u] = ld_quad((const Quad*)data + q);
                    uint32_t c[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        c[e] = !((m[u] >> (8 * e)) & 0xffu) ? 0u
                             : LUT ? s_lut[(uint8_t)a[u].v[e]] : colour_of(p, ValT<KIND>::get(a[u].v[e]));
                    out = make_uint4(c[0], c[1], c[2], c[3]);
                }
                st_stream((uint4*)rgba + q, out);
            }
        }
        done = nq << 2;
    }
    for (long long i = done + tid; i < n; i += nthreads)
        rgba[i] = !mask[i] ? 0u : LUT ? s_lut[(uint8_t)data[i]] : colour_of(p, ValT<KIND>::get(data[i]));
}

// 16 mask bytes -> 2 packed bytes per thread
__global__ void __launch_bounds__(BLOCK)
pack_kernel(const uint8_t* __restrict__ mask, long long n, uint8_t* __restrict__ bits) {
    const long long nthreads = (long long)gridDim.x * BLOCK;
    const long long nbytes = (n + 7) >> 3;
    const bool vec = (((uintptr_t)mask) & 7) == 0;
    for (long long b = (long long)blockIdx.x * BLOCK + threadIdx.x; b < nbytes; b += nthreads) {
        unsigned out = 0;
        const long long i0 = b << 3;
        if (vec && i0 + 8 <= n) {
            const uint2 w = *(const uint2*)(mask + i0);
            const unsigned lo = nz_bits4(w.x), hi = nz_bits4(w.y);    // bit e <-> byte e
            const unsigned byte = lo | (hi << 4);                     // bit j <-> texel i0 + j
            out = __brev(byte) >> 24;                                 // MSB first
        } else {
            for (int j = 0; j < 8; ++j) if (i0 + j < n && mask[i0 + j]) out |= 0x80u >> j;
        }
        bits[b] = (uint8_t)out;
    }
}

// 2 packed bytes -> 16 mask bytes (one 128-bit store) per thread; scalar tail / unaligned planes
__global__ void __launch_bounds__(BLOCK)
unpack_kernel(const uint8_t* __restrict__ bits, long long n, uint8_t* __restrict__ mask) {
    const long long nthreads = (long long)gridDim.x * BLOCK;
    const long long tid = (long long)blockIdx.x * BLOCK + threadIdx.x;
    long long done = 0;
    if (((((uintptr_t)mask) & 15) | (((uintptr_t)bits) & 1)) == 0) {
        const long long nv = n >> 4;
        for (long long v = tid; v < nv; v += nthreads) {
            const unsigned two = *(const uint16_t*)(bits + 2 * v);             // byte 0 = texels 0..7 (MSB first)
            uint32_t w[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const unsigned nib = ((two >> (8 * (k >> 1))) >> ((k & 1) ? 0 : 4)) & 0xfu;   // 4 texels, MSB = first
                w[k] = ((nib >> 3) & 1u) | (((nib >> 2) & 1u) << 8) | (((nib >> 1) & 1u) << 16) | ((nib & 1u) << 24);
            }
            st_stream((uint4*)mask + v, make_uint4(w[0], w[1], w[2], w[3]));
        }
        done = nv << 4;
    }
    for (long long i = done + tid; i < n; i += nthreads)
        mask[i] = (bits[i >> 3] >> (7 - (i & 7))) & 1u;
}

inline unsigned grid_for(long long items) {
    long long blocks = (items + BLOCK - 1) / BLOCK;
    const long long cap = (long long)ml_sm_count() * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (unsigned)blocks;
}

template <int KIND>
int launch_display(const void* data, const uint8_t* mask, long long n, const PaletteArgs& p, uint32_t* rgba, cudaStream_t st) {
    display_kernel<KIND><<<grid_for((n + 15) >> 4), BLOCK, 0, st>>>(data, mask, n, p, rgba);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

}  // namespace

extern "C" {

int ml_resolve_display(const void* data, int kind, const uint8_t* mask, int64_t n,
                       double lower, double upper, const double* positions, const double* rgba_points,
                       int npoints, uint8_t* rgba_out, void* stream) {
    if (npoints < 2 || npoints > MAX_POINTS) return ml_fail(ML_ERR_ARG, "palette needs 2..64 control points");
    if (!(lower < upper)) return ml_fail(ML_ERR_ARG, "display limits need lower < upper");
    if (n <= 0) return ML_OK;
    PaletteArgs p;
    p.npoints = npoints; p.lower = lower; p.upper = upper;
    for (int k = 0; k < npoints; ++k) {
        p.pos[k] = positions[k];
        for (int c = 0; c < 4; ++c) p.rgba[k][c] = rgba_points[4 * k + c];
        if (k > 0 && !(positions[k] > positions[k - 1])) return ml_fail(ML_ERR_ARG, "palette positions must increase");
    }
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t* out = (uint32_t*)rgba_out;
    switch (kind) {
    case ML_U8:  return launch_display<ML_U8>(data, mask, n, p, out, st);
    case ML_I8:  return launch_display<ML_I8>(data, mask, n, p, out, st);
    case ML_I16: return launch_display<ML_I16>(data, mask, n, p, out, st);
    case ML_I32: return launch_display<ML_I32>(data, mask, n, p, out, st);
    case ML_U32: return launch_display<ML_U32>(data, mask, n, p, out, st);
    case ML_F16: return launch_display<ML_F16>(data, mask, n, p, out, st);
    case ML_FLOAT32: return launch_display<ML_FLOAT32>(data, mask, n, p, out, st);
    }
    return ml_fail(ML_ERR_ARG, "unknown plane kind");
}

int ml_pack_mask(const uint8_t* mask, int64_t n, uint8_t* bits, void* stream) {
    if (n <= 0) return ML_OK;
    pack_kernel<<<grid_for((n + 7) >> 3), BLOCK, 0, (cudaStream_t)stream>>>(mask, n, bits);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int ml_unpack_mask(const uint8_t* bits, int64_t n, uint8_t* mask, void* stream) {
    if (n <= 0) return ML_OK;
    unpack_kernel<<<grid_for((n + 15) >> 4), BLOCK, 0, (cudaStream_t)stream>>>(bits, n, mask);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

}  // extern "C"
