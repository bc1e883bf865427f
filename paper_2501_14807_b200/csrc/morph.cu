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
#include "common.cuh"
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
    padding_kernel<<<grid_for(((width + 3) >> 2) * out_rows), BLOCK, 0, (cudaStream_t)stream>>>(
        outline, edited, width, in_row0, in_rows, out_row0, out_rows, (int)radius, data, esize,
        value_bits, mask, (unsigned long long*)count);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

}  // extern "C"
