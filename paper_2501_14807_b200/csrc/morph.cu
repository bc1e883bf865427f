// Texture Padding Algorithm (TPA) stencils: outline mask and padding (SPEC.md:286-303,
// PAPER.md section 4.3.2).  Chebyshev (box) neighbourhoods.  Frozen definitions:
// oracle/kn_port.c ext_outline / ext_padding; known answers SPEC.md:293, 298, 608.
//
// Row-sharded use: the INPUT plane is a slab of global rows [in_row0, in_row0+in_rows) that must
// include the `radius` halo rows a rank can see; rows outside the slab count as empty.  The
// OUTPUT planes are slabs of rows [out_row0, out_row0+out_rows).
//
// Each thread produces 4 horizontally adjacent texels: for every neighbour row it scans the
// bytes [x-r, x+3+r] once and derives the four windows from a running byte mask, so the stencil
// costs (2r+1)*(4+2r) byte reads per 4 texels, served from L1/L2.
#include <stdlib.h>
#include "common.cuh"
#include "bulk.cuh"
#include "meshlayers_b200.h"
#include "internal.h"

namespace {

constexpr int BLOCK = 256;

// bit e of the result: some byte of src row segment [x+e-r, x+e+r] (clipped to [0,width)) is != 0
ML_DEV unsigned row_windows(const uint8_t* __restrict__ row, long long width, long long x, int r) {
    unsigned res = 0;
    // nz bit j <-> byte at column x - r + j, j in [0, 4+2r)
    unsigned long long nz = 0;
    const int span = 4 + 2 * r;
    if (span <= 64) {
        for (int j = 0; j < span; ++j) {
            const long long c = x - r + j;
            if (c >= 0 && c < width && row[c] != 0) nz |= 1ull << j;
        }
        const unsigned long long win = (span >= 64 + 4) ? ~0ull : ((1ull << (2 * r + 1)) - 1ull);
#pragma unroll
        for (int e = 0; e < 4; ++e) if (nz & (win << e)) res |= 1u << e;
    } else {
        for (int e = 0; e < 4; ++e)
            for (int j = -r; j <= r; ++j) {
                const long long c = x + e + j;
                if (c >= 0 && c < width && row[c] != 0) { res |= 1u << e; break; }
            }
    }
    return res;
}

// near[e] for the 4 texels starting at (x, y): any src != 0 within Chebyshev distance r
ML_DEV unsigned box_any(const uint8_t* __restrict__ src, long long width, long long in_row0,
                        long long in_rows, long long x, long long y, int r) {
    unsigned res = 0;
    for (long long yy = y - r; yy <= y + r && res != 0xfu; ++yy) {
        if (yy < in_row0 || yy >= in_row0 + in_rows) continue;
        res |= row_windows(src + (yy - in_row0) * width, width, x, r);
    }
    return res;
}

__global__ void __launch_bounds__(BLOCK)
outline_kernel(const uint8_t* __restrict__ cov, long long width, long long in_row0, long long in_rows,
               long long out_row0, long long out_rows, int r, uint8_t* __restrict__ outline) {
    const long long qw = (width + 3) >> 2;                 // quads per row
    const long long nq = qw * out_rows;
    const long long nthreads = (long long)gridDim.x * BLOCK;
    for (long long q = (long long)blockIdx.x * BLOCK + threadIdx.x; q < nq; q += nthreads) {
        const long long yy = q / qw, x = (q - yy * qw) << 2, y = out_row0 + yy;
        const uint8_t* crow = cov + (y - in_row0) * width;
        unsigned uncovered = 0;
        for (int e = 0; e < 4; ++e) if (x + e < width && crow[x + e] == 0) uncovered |= 1u << e;
        unsigned near = uncovered ? box_any(cov, width, in_row0, in_rows, x, y, r) : 0u;
        for (int e = 0; e < 4; ++e)
            if (x + e < width) outline[yy * width + x + e] = ((uncovered & near) >> e) & 1u;
    }
}

__global__ void __launch_bounds__(BLOCK)
padding_kernel(const uint8_t* __restrict__ outline, const uint8_t* __restrict__ edited, long long width,
               long long in_row0, long long in_rows, long long out_row0, long long out_rows, int r,
               void* __restrict__ data, int esize, uint32_t value, uint8_t* __restrict__ mask,
               unsigned long long* count) {
    const long long qw = (width + 3) >> 2;
    const long long nq = qw * out_rows;
    const long long nthreads = (long long)gridDim.x * BLOCK;
    long long cnt = 0;
    for (long long q = (long long)blockIdx.x * BLOCK + threadIdx.x; q < nq; q += nthreads) {
        const long long yy = q / qw, x = (q - yy * qw) << 2, y = out_row0 + yy;
        unsigned on = 0;
        for (int e = 0; e < 4; ++e) if (x + e < width && outline[yy * width + x + e] != 0) on |= 1u << e;
        if (!on) continue;
        const unsigned near = box_any(edited, width, in_row0, in_rows, x, y, r);
        const unsigned hit = on & near;
        for (int e = 0; e < 4; ++e)
            if (hit & (1u << e)) {
                const long long i = yy * width + x + e;
                store_value(data, esize, i, value);
                mask[i] = 1;
                ++cnt;
            }
    }
    block_count_add(cnt, count);
}

// 4-bit mask of the non-zero byte lanes of a 32-bit word
ML_DEV unsigned nz4(uint32_t w) { return nz_bits4(w); }

// 16-bit mask: texel x0+e (x0 % 16 == 0) has some src != 0 within Chebyshev distance r <= 4.
// Per neighbour row THREE independent aligned loads (word left, 16-byte vector, word right) give
// the non-zero bits of columns [x0-4, x0+20); all rows' loads are in flight together, then the
// windows are a bit dilation.  (The byte-at-a-time box_any costs (2r+1)(4+2r) dependent L2
// accesses per 4 texels, which made thin outline columns dominate the pass.)
ML_DEV unsigned box_any16(const uint8_t* __restrict__ src, long long width, long long in_row0,
                          long long in_rows, long long x0, long long y, int r) {
    unsigned bits = 0;                                    // bit j <-> column x0 - 4 + j
    for (int dy = -r; dy <= r; ++dy) {
        const long long yy = y + dy;
        if (yy < in_row0 || yy >= in_row0 + in_rows) continue;
        const uint8_t* row = src + (yy - in_row0) * width + x0;
        const uint4 c = *(const uint4*)row;
        const uint32_t l = x0 >= 4 ? *(const uint32_t*)(row - 4) : 0u;
        const uint32_t rr = x0 + 16 < width ? *(const uint32_t*)(row + 16) : 0u;
        bits |= nz4(l) | (nz4(c.x) << 4) | (nz4(c.y) << 8) | (nz4(c.z) << 12) | (nz4(c.w) << 16) | (nz4(rr) << 20);
    }
    unsigned d = bits;
    for (int k = 1; k <= r; ++k) d |= (bits << k) | (bits >> k);
    return (d >> 4) & 0xffffu;
}

// Streaming form of the padding pass for the per-stroke hot path (width % 16 == 0, 16-byte
// aligned planes, radius <= 4): the outline plane is the 1 B/texel read stream (four 128-bit loads
// in flight per thread); outlines are thin, so almost every 16-texel vector is all zero and is
// skipped; vectors with outline texels fetch their neighbourhood of the edited plane with
// 3*(2r+1) independent loads.  Data / mask are updated with 32-bit read-modify-writes (each
// 4-texel word is owned by one thread).
// Outline mask, 16 texels per thread (width % 16 == 0, 16-byte aligned planes, thickness <= 4): the
// coverage vector is one 128-bit load; fully covered vectors (the bulk of an atlas) store zeros at
// once, the others get the covered-neighbourhood bits from box_any16 (3 aligned loads per row).
__global__ void __launch_bounds__(BLOCK)
outline_vec_kernel(const uint8_t* __restrict__ cov, long long width, long long in_row0, long long in_rows,
                   long long out_row0, long long out_rows, int r, uint8_t* __restrict__ outline) {
    const long long nv = (width * out_rows) >> 4;
    const long long nthreads = (long long)gridDim.x * BLOCK;
    for (long long v = (long long)blockIdx.x * BLOCK + threadIdx.x; v < nv; v += nthreads) {
        const long long i0 = v << 4;
        const long long yy = i0 / width, x0 = i0 - yy * width, y = out_row0 + yy;
        const uint4 c = ld_stream((const uint4*)(cov + (y - in_row0) * width + x0));
        const unsigned covered = nz4(c.x) | (nz4(c.y) << 4) | (nz4(c.z) << 8) | (nz4(c.w) << 12);
        unsigned out16 = 0;
        if (covered != 0xffffu) out16 = ~covered & 0xffffu & box_any16(cov, width, in_row0, in_rows, x0, y, r);
        uint4 o;
        o.x = spread4(out16 & 0xfu) & 0x01010101u;         o.y = spread4((out16 >> 4) & 0xfu) & 0x01010101u;
        o.z = spread4((out16 >> 8) & 0xfu) & 0x01010101u;  o.w = spread4((out16 >> 12) & 0xfu) & 0x01010101u;
        st_stream((uint4*)(outline + i0), o);
    }
}

// One 16-texel vector of the padding pass: `o` = its outline bytes (non-zero somewhere), i0 = flat
// index of its first texel.  Returns the number of padded texels.
template <int ES>
ML_DEV int pad_vector(const uint4& o, long long i0, const uint8_t* __restrict__ edited, long long width,
                      long long in_row0, long long in_rows, long long out_row0, int r,
                      void* __restrict__ data, uint32_t value, uint8_t* __restrict__ mask) {
    const long long yy = i0 / width, x0 = i0 - yy * width;
    const unsigned on = nz4(o.x) | (nz4(o.y) << 4) | (nz4(o.z) << 8) | (nz4(o.w) << 12);
    const unsigned hit16 = on & box_any16(edited, width, in_row0, in_rows, x0, out_row0 + yy, r);
    if (!hit16) return 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const unsigned hit = (hit16 >> (4 * j)) & 0xfu;
        if (!hit) continue;
        const long long i = i0 + 4 * j;
        const uint32_t hm = spread4(hit);
        uint32_t* pm = (uint32_t*)(mask + i);
        const uint32_t mw = *pm, mn = (mw & ~hm) | (0x01010101u & hm);
        if (mn != mw) *pm = mn;
        if (ES == 1) {
            uint32_t* pd = (uint32_t*)((uint8_t*)data + i);
            const uint32_t dw = *pd;
            *pd = (dw & ~hm) | (((value & 0xffu) * 0x01010101u) & hm);
        } else if (ES == 2) {
#pragma unroll
            for (int e = 0; e < 4; ++e) if (hit & (1u << e)) ((uint16_t*)data)[i + e] = (uint16_t)value;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) if (hit & (1u << e)) ((uint32_t*)data)[i + e] = value;
        }
    }
    return __popc(hit16);
}

// Streaming form of the padding pass for the per-stroke hot path (width % 16 == 0, 16-byte
// aligned planes, radius <= 4): the outline plane is the 1 B/texel read stream (four 128-bit loads
// in flight per thread); outlines are thin, so almost every 16-texel vector is all zero and is
// skipped; vectors with outline texels fetch their neighbourhood of the edited plane with
// 3*(2r+1) independent loads.  Data / mask are updated with 32-bit read-modify-writes (each
// 4-texel word is owned by one thread).
template <int ES>
__global__ void __launch_bounds__(BLOCK)
padding_stream_kernel(const uint8_t* __restrict__ outline, const uint8_t* __restrict__ edited, long long width,
                      long long in_row0, long long in_rows, long long out_row0, long long out_rows, int r,
                      void* __restrict__ data, uint32_t value, uint8_t* __restrict__ mask,
                      unsigned long long* count) {
    constexpr int U = 4;
    const long long nv = (width * out_rows) >> 4;
    const long long tid = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * BLOCK;
    long long cnt = 0;
    for (long long v0 = tid; v0 < nv; v0 += nthreads * U) {
        uint4 o[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long v = v0 + u * nthreads;
            o[u] = v < nv ? ld_stream((const uint4*)outline + v) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll 1
        for (int u = 0; u < U; ++u) {
            if ((o[u].x | o[u].y | o[u].z | o[u].w) == 0) continue;
            cnt += pad_vector<ES>(o[u], (v0 + u * nthreads) << 4, edited, width, in_row0, in_rows, out_row0, r, data, value, mask);
        }
    }
    block_count_add(cnt, count);
}

// Bulk-copy form of the streaming padding pass (the default for aligned planes): the outline plane
// -- the kernel's whole 1 B/texel read stream -- is fetched by ONE producer lane per block with
// cp.async.bulk into a PAD_STAGES x PAD_CHUNK shared-memory ring (bulk.cuh); the eight consumer warps
// read their two 16-texel vectors of a chunk with conflict-free 128-bit LDS, release the stage and
// only then look at the (rare) vectors that hold outline texels.  The register form above keeps
// 64 B per thread in flight and stalls the whole block behind its slowest load (ncu r1: 28 % of the
// DRAM peak, barrier + long-scoreboard stalls); here blocks/SM x PAD_STAGES x 8 KB are in flight
// whatever the consumers are doing.
#ifndef ML_PAD_STAGES
#define ML_PAD_STAGES 4
#endif
constexpr int PAD_STAGES = ML_PAD_STAGES;
constexpr int PAD_CHUNK = 8192;                       // bytes == texels per chunk
constexpr int PAD_CONSUMER_WARPS = 8;
constexpr int PAD_THREADS = 32 * (PAD_CONSUMER_WARPS + 1);
constexpr int PAD_VPT = PAD_CHUNK / (16 * 32 * PAD_CONSUMER_WARPS);     // 16-texel vectors per consumer thread and chunk
typedef BulkRing<PAD_STAGES, PAD_CHUNK> PadRing;

// Vectors that hold outline texels are rare (an outline is a thin curve) but expensive: their
// 3 x (2r+1) neighbourhood loads of `edited` are a dependent DRAM round trip.  Handled in place
// they serialise the stream behind one lane per chunk (ncu r2: long_scoreboard 19.9 per issue, 37 %
// of the DRAM peak -- the left / right island border puts one such vector into EVERY chunk, always
// in the same warp).  Instead each warp queues the vector indices in shared memory and, once 32 are
// waiting (and at the end), processes them one per lane, so 32 neighbourhood fetches overlap.
constexpr int PAD_QCAP = 64;                          // queue slots per consumer warp (flushed at >= 32)

template <int ES>
ML_DEV long long pad_flush(long long* q, int count, int lane, const uint8_t* __restrict__ outline,
                           const uint8_t* __restrict__ edited, long long width, long long in_row0, long long in_rows,
                           long long out_row0, int r, void* __restrict__ data, uint32_t value, uint8_t* __restrict__ mask) {
    long long cnt = 0;
    __syncwarp();
    if (lane < count) {
        const long long i0 = q[lane];
        const uint4 o = *(const uint4*)(outline + i0);
        cnt = pad_vector<ES>(o, i0, edited, width, in_row0, in_rows, out_row0, r, data, value, mask);
    }
    __syncwarp();
    return cnt;
}

template <int ES>
__global__ void __launch_bounds__(PAD_THREADS)
padding_bulk_kernel(const uint8_t* __restrict__ outline, const uint8_t* __restrict__ edited, long long width,
                    long long in_row0, long long in_rows, long long out_row0, long long out_rows, int r,
                    void* __restrict__ data, uint32_t value, uint8_t* __restrict__ mask,
                    unsigned long long* count) {
    extern __shared__ __align__(128) uint8_t pad_smem[];
    PadRing& ring = *reinterpret_cast<PadRing*>(pad_smem);
    __shared__ long long s_queue[PAD_CONSUMER_WARPS][PAD_QCAP];
    const long long n = width * out_rows;                  // multiple of 16 (host checks width % 16 == 0)
    const long long nchunks = (n + PAD_CHUNK - 1) / PAD_CHUNK;
    if (threadIdx.x == 0) ring.init(PAD_CONSUMER_WARPS);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    long long cnt = 0;
    RingPos<PAD_STAGES> pos;
    if (warp == PAD_CONSUMER_WARPS) {
        if (lane == 0) {
            const uint64_t policy = l2_policy_evict_first();
            for (long long c = blockIdx.x; c < nchunks; c += gridDim.x, pos.next()) {
                const long long base = c * PAD_CHUNK;
                const unsigned bytes = (unsigned)(n - base < PAD_CHUNK ? n - base : PAD_CHUNK);
                ring.produce(pos, outline + base, bytes, policy);
            }
        }
    } else {
        long long* q = s_queue[warp];
        int queued = 0;                                    // warp-uniform
        for (long long c = blockIdx.x; c < nchunks; c += gridDim.x, pos.next()) {
            const long long base = c * PAD_CHUNK;
            const unsigned bytes = (unsigned)(n - base < PAD_CHUNK ? n - base : PAD_CHUNK);
            const uint8_t* b = ring.acquire(pos);
            bool nz[PAD_VPT];
#pragma unroll
            for (int u = 0; u < PAD_VPT; ++u) {
                const unsigned off = (unsigned)(u * 32 * PAD_CONSUMER_WARPS + threadIdx.x) << 4;
                uint4 o = make_uint4(0, 0, 0, 0);
                if (off < bytes) o = *(const uint4*)(b + off);
                nz[u] = (o.x | o.y | o.z | o.w) != 0;
            }
            ring.release(pos);
#pragma unroll
            for (int u = 0; u < PAD_VPT; ++u) {
                const unsigned bal = __ballot_sync(0xffffffffu, nz[u]);
                if (bal == 0) continue;
                if (nz[u]) q[queued + __popc(bal & ((1u << lane) - 1u))] = base + ((unsigned)(u * 32 * PAD_CONSUMER_WARPS + threadIdx.x) << 4);
                queued += __popc(bal);
                if (queued >= 32) {
                    cnt += pad_flush<ES>(q, 32, lane, outline, edited, width, in_row0, in_rows, out_row0, r, data, value, mask);
                    if (lane < queued - 32) q[lane] = q[32 + lane];       // <= 32 left over: move to the front
                    queued -= 32;
                    __syncwarp();
                }
            }
        }
        if (queued) cnt += pad_flush<ES>(q, queued, lane, outline, edited, width, in_row0, in_rows, out_row0, r, data, value, mask);
    }
    block_count_add(cnt, count);
}

// Footprint-culled form (single slab, width % 128 == 0, radius <= 4): `tile_bits` is the bitmap of
// 128 x 8-texel tiles the TEA stroke could edit (ml_tea_classify).  A padded texel lies within
// `radius` <= 4 texels of an edited one, i.e. in a marked tile or one of its 8 neighbours, so one
// warp per tile tests the 3 x 3 tile neighbourhood in the bitmap and reads the outline bytes of
// that tile only when some neighbour is marked.  Same planes and count as the streaming kernel.
template <int ES>
__global__ void __launch_bounds__(BLOCK)
padding_tile_kernel(const uint8_t* __restrict__ outline, const uint8_t* __restrict__ edited, long long width,
                    long long rows, long long row_lo, long long row_hi, int r, const uint32_t* __restrict__ tile_bits,
                    void* __restrict__ data, uint32_t value, uint8_t* __restrict__ mask, unsigned long long* count) {
    __shared__ int s_list[BLOCK];
    __shared__ int s_n;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int segs = (int)(width >> 7);
    const int tile_rows = (int)((rows + 7) >> 3);
    const int ntiles = segs * tile_rows;
    long long cnt = 0;
    // each thread tests ONE tile's 3 x 3 neighbourhood; the block compacts the tiles to visit into
    // shared memory and its warps share them (the marked tiles of a stroke are clustered)
    for (int base = blockIdx.x * BLOCK; base < ntiles; base += gridDim.x * BLOCK) {
        if (threadIdx.x == 0) s_n = 0;
        __syncthreads();
        const int tile = base + threadIdx.x;
        bool near = false;
        if (tile < ntiles) {
            const int ty = tile / segs, tx = tile - ty * segs;
#pragma unroll
            for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                for (int dx = -1; dx <= 1; ++dx) {
                    const int y = ty + dy, x = tx + dx;
                    if (y < 0 || y >= tile_rows || x < 0 || x >= segs) continue;
                    const int t = y * segs + x;
                    near |= ((__ldg(tile_bits + (t >> 5)) >> (t & 31)) & 1u) != 0;
                }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, near);
        int off = 0;
        if (lane == 0 && bal) off = atomicAdd(&s_n, __popc(bal));
        off = __shfl_sync(0xffffffffu, off, 0);
        if (near) s_list[off + __popc(bal & ((1u << lane) - 1u))] = tile;
        __syncthreads();
        const int nlist = s_n;
        for (int j = wid; j < nlist; j += BLOCK / 32) {
            const int t = s_list[j];
            const int ty = t / segs, tx = t - ty * segs;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int v = lane + 32 * k;                   // 64 vectors of 16 texels per tile
                const long long yy = ((long long)ty << 3) + (v >> 3);
                if (yy < row_lo || yy >= row_hi) continue;     // rows outside [row_lo, row_hi) belong to the caller's border pass
                const long long i0 = yy * width + ((long long)tx << 7) + ((v & 7) << 4);
                const uint4 o = ld_stream((const uint4*)(outline + i0));
                if ((o.x | o.y | o.z | o.w) == 0) continue;
                cnt += pad_vector<ES>(o, i0, edited, width, 0, rows, 0, r, data, value, mask);
            }
        }
        __syncthreads();
    }
    block_count_add(cnt, count);
}

inline unsigned grid_for(long long items) {
    long long blocks = (items + BLOCK - 1) / BLOCK;
    const long long cap = (long long)ml_sm_count() * 32;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (unsigned)blocks;
}

}  // namespace

extern "C" {

int ml_outline_mask(const uint8_t* cov, int64_t width, int64_t in_row0, int64_t in_rows,
                    int64_t out_row0, int64_t out_rows, int64_t thickness, uint8_t* outline,
                    void* stream) {
    if (thickness < 0 || thickness > 1 << 20) return ml_fail(ML_ERR_ARG, "bad outline thickness");
    if (out_row0 < in_row0 || out_row0 + out_rows > in_row0 + in_rows)
        return ml_fail(ML_ERR_ARG, "output rows must lie inside the input slab");
    if (out_rows <= 0 || width <= 0) return ML_OK;
    if ((width % 16) == 0 && thickness >= 1 && thickness <= 4 && ((((uintptr_t)cov) | ((uintptr_t)outline)) & 15) == 0)
        outline_vec_kernel<<<grid_for((width * out_rows) >> 4), BLOCK, 0, (cudaStream_t)stream>>>(
            cov, width, in_row0, in_rows, out_row0, out_rows, (int)thickness, outline);
    else
        outline_kernel<<<grid_for(((width + 3) >> 2) * out_rows), BLOCK, 0, (cudaStream_t)stream>>>(
            cov, width, in_row0, in_rows, out_row0, out_rows, (int)thickness, outline);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int ml_apply_padding(const uint8_t* outline, const uint8_t* edited, int64_t width,
                     int64_t in_row0, int64_t in_rows, int64_t out_row0, int64_t out_rows,
                     int64_t radius, void* data, int esize, uint32_t value_bits, uint8_t* mask,
                     uint64_t* count, void* stream) {
    if (esize != 1 && esize != 2 && esize != 4) return ml_fail(ML_ERR_ARG, "esize must be 1, 2 or 4");
    if (radius > 1 << 20) return ml_fail(ML_ERR_ARG, "bad padding radius");
    if (out_row0 < in_row0 || out_row0 + out_rows > in_row0 + in_rows)
        return ml_fail(ML_ERR_ARG, "output rows must lie inside the input slab");
    if (radius <= 0 || out_rows <= 0 || width <= 0) return ML_OK;      /* SPEC.md:303 radius 0 -> nothing */
    const bool vec = (width % 16 == 0) && radius <= 4 &&
                     ((((uintptr_t)outline) | ((uintptr_t)edited) | ((uintptr_t)data) | ((uintptr_t)mask)) & 15) == 0;
    if (vec) {
        const long long nv = (width * out_rows) >> 4;
        long long blocks = (nv + (long long)BLOCK * 4 - 1) / ((long long)BLOCK * 4);
        const long long cap = (long long)ml_sm_count() * 16;
        if (blocks > cap) blocks = cap;
        if (blocks < 1) blocks = 1;
        cudaStream_t st = (cudaStream_t)stream;
        static const bool reg_form = getenv("ML_PAD_REGISTER_STREAM") != nullptr;       // the round-1 kernel, kept for comparison
        if (!reg_form && nv * 16 >= 4 * PAD_CHUNK) {
            static int per_sm[3] = {0, 0, 0};
            const int k = esize == 1 ? 0 : (esize == 2 ? 1 : 2);
            const void* fn = esize == 1 ? (const void*)padding_bulk_kernel<1> : (esize == 2 ? (const void*)padding_bulk_kernel<2> : (const void*)padding_bulk_kernel<4>);
            if (!per_sm[k]) {
                ML_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PadRing)));
                int nb = 0;
                ML_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, PAD_THREADS, sizeof(PadRing)));
                per_sm[k] = nb > 0 ? nb : 1;
            }
            const long long nchunks = (nv * 16 + PAD_CHUNK - 1) / PAD_CHUNK;
            long long g = (long long)ml_sm_count() * per_sm[k];
            if (g > nchunks) g = nchunks;
#define ML_LAUNCH_PADB(ES) padding_bulk_kernel<ES><<<(unsigned)g, PAD_THREADS, sizeof(PadRing), st>>>(outline, edited, width, in_row0, in_rows, out_row0, out_rows, (int)radius, data, value_bits, mask, (unsigned long long*)count)
            if (esize == 1) ML_LAUNCH_PADB(1); else if (esize == 2) ML_LAUNCH_PADB(2); else ML_LAUNCH_PADB(4);
#undef ML_LAUNCH_PADB
            ML_CUDA(cudaGetLastError());
            return ML_OK;
        }
#define ML_LAUNCH_PAD(ES) padding_stream_kernel<ES><<<(unsigned)blocks, BLOCK, 0, st>>>(outline, edited, width, in_row0, in_rows, out_row0, out_rows, (int)radius, data, value_bits, mask, (unsigned long long*)count)
        if (esize == 1) ML_LAUNCH_PAD(1); else if (esize == 2) ML_LAUNCH_PAD(2); else ML_LAUNCH_PAD(4);
#undef ML_LAUNCH_PAD
        ML_CUDA(cudaGetLastError());
        return ML_OK;
    }
    padding_kernel<<<grid_for(((width + 3) >> 2) * out_rows), BLOCK, 0, (cudaStream_t)stream>>>(
        outline, edited, width, in_row0, in_rows, out_row0, out_rows, (int)radius, data, esize,
        value_bits, mask, (unsigned long long*)count);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int ml_apply_padding_tiles(const uint8_t* outline, const uint8_t* edited, int64_t width, int64_t rows,
                           int64_t radius, const uint32_t* tile_bits, void* data, int esize,
                           uint32_t value_bits, uint8_t* mask, uint64_t* count, void* stream) {
    return ml_apply_padding_tiles_rows(outline, edited, width, rows, 0, rows, radius, tile_bits, data, esize,
                                       value_bits, mask, count, stream);
}

int ml_apply_padding_tiles_rows(const uint8_t* outline, const uint8_t* edited, int64_t width, int64_t rows,
                                int64_t row_lo, int64_t row_hi, int64_t radius, const uint32_t* tile_bits,
                                void* data, int esize, uint32_t value_bits, uint8_t* mask, uint64_t* count,
                                void* stream) {
    if (esize != 1 && esize != 2 && esize != 4) return ml_fail(ML_ERR_ARG, "esize must be 1, 2 or 4");
    if (row_lo < 0) row_lo = 0;
    if (row_hi > rows) row_hi = rows;
    if (radius <= 0 || rows <= 0 || width <= 0 || row_lo >= row_hi) return ML_OK;
    if ((width % 128) != 0 || radius > 4 || tile_bits == nullptr ||
        ((((uintptr_t)outline) | ((uintptr_t)edited) | ((uintptr_t)data) | ((uintptr_t)mask)) & 15) != 0)
        return ml_fail(ML_ERR_ARG, "culled padding needs width % 128 == 0, radius <= 4, aligned planes and the stroke's tile bitmap");
    const long long ntiles = (width >> 7) * ((rows + 7) >> 3);
    long long blocks = (ntiles + BLOCK - 1) / BLOCK;               // one tile per thread in the classification step
    const long long cap = (long long)ml_sm_count() * 8;
    if (blocks > cap) blocks = cap;
    cudaStream_t st = (cudaStream_t)stream;
#define ML_LAUNCH_PADT(ES) padding_tile_kernel<ES><<<(unsigned)blocks, BLOCK, 0, st>>>(outline, edited, width, rows, row_lo, row_hi, (int)radius, tile_bits, data, value_bits, mask, (unsigned long long*)count)
    if (esize == 1) ML_LAUNCH_PADT(1); else if (esize == 2) ML_LAUNCH_PADT(2); else ML_LAUNCH_PADT(4);
#undef ML_LAUNCH_PADT
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

}  // extern "C"
