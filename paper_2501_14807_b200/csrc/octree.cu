// Octree baseline kernels -- the other two callables of the reference's
// compiled-backend slot: expand_pairs_ordered (KN:303-329, triangle / box separating-axis test,
// KN:208-258) and raycast (KN:361-525, 3D-DDA over the Morton-keyed leaf grid with
// Moeller-Trumbore, KN:335-358).  Both are bit-exact restatements: float64, the reference's
// association order, no contraction (the library is compiled with -fmad=false, build.py), and
// np.minimum / np.maximum semantics (NaN propagates).
//
// Work decomposition
//   expand : one thread per (pair, octant) -- the 8 lanes of a pair read the same triangle
//            (broadcast loads) and thread order == output order (pair-major, octant-minor), so a
//            ballot gives every hit its output slot.  Pass 1 writes one hit byte per pair and
//            one total per 1024-pair chunk, a single-block scan turns the totals into offsets,
//            pass 2 re-reads the hit bytes (not the geometry) and emits.
//   raycast: one thread per ray (nothing couples two rays: the reference's lexsort, KN:474-487,
//            is a per-ray lexicographic minimum over (t, triangle index)); the coarse occupancy
//            map and the sorted key array are read through L1/L2.
#include "internal.h"

namespace {

constexpr int EXP_THREADS = 256;                 // 32 pairs per block step
constexpr int EXP_CHUNK = 1024;                  // pairs per block

ML_DEV double np_min(double a, double b) { return (a != a) ? a : ((b != b) ? b : (a < b ? a : b)); }
ML_DEV double np_max(double a, double b) { return (a != a) ? a : ((b != b) ? b : (a > b ? a : b)); }
ML_DEV double min3(double a, double b, double c) { return np_min(np_min(a, b), c); }
ML_DEV double max3(double a, double b, double c) { return np_max(np_max(a, b), c); }

// KN:208-258: vertices relative to the cell centre, h = half extent; true = separated
ML_DEV bool sat_separated(const double vx[3], const double vy[3], const double vz[3], double h) {
    bool sep = (min3(vx[0], vx[1], vx[2]) > h) | (max3(vx[0], vx[1], vx[2]) < -h);
    sep |= (min3(vy[0], vy[1], vy[2]) > h) | (max3(vy[0], vy[1], vy[2]) < -h);
    sep |= (min3(vz[0], vz[1], vz[2]) > h) | (max3(vz[0], vz[1], vz[2]) < -h);
    double ex[3], ey[3], ez[3];
    ex[0] = vx[1] - vx[0]; ey[0] = vy[1] - vy[0]; ez[0] = vz[1] - vz[0];
    ex[1] = vx[2] - vx[1]; ey[1] = vy[2] - vy[1]; ez[1] = vz[2] - vz[1];
    ex[2] = vx[0] - vx[2]; ey[2] = vy[0] - vy[2]; ez[2] = vz[0] - vz[2];
    const double nx = ey[0] * ez[1] - ez[0] * ey[1];                 // KN:229-231
    const double ny = ez[0] * ex[1] - ex[0] * ez[1];
    const double nz = ex[0] * ey[1] - ey[0] * ex[1];
    double r = h * ((fabs(nx) + fabs(ny)) + fabs(nz));
    const double d = (nx * vx[0] + ny * vy[0]) + nz * vz[0];
    sep |= (d > r) | (d < -r);
#pragma unroll
    for (int k = 0; k < 3; ++k) {                                    // KN:236-257
        double p0, p1, p2;
        r = h * (fabs(ez[k]) + fabs(ey[k]));
        p0 = ez[k] * vy[0] - ey[k] * vz[0];
        p1 = ez[k] * vy[1] - ey[k] * vz[1];
        p2 = ez[k] * vy[2] - ey[k] * vz[2];
        sep |= (min3(p0, p1, p2) > r) | (max3(p0, p1, p2) < -r);
        r = h * (fabs(ez[k]) + fabs(ex[k]));
        p0 = ex[k] * vz[0] - ez[k] * vx[0];
        p1 = ex[k] * vz[1] - ez[k] * vx[1];
        p2 = ex[k] * vz[2] - ez[k] * vx[2];
        sep |= (min3(p0, p1, p2) > r) | (max3(p0, p1, p2) < -r);
        r = h * (fabs(ey[k]) + fabs(ex[k]));
        p0 = ey[k] * vx[0] - ex[k] * vy[0];
        p1 = ey[k] * vx[1] - ex[k] * vy[1];
        p2 = ey[k] * vx[2] - ex[k] * vy[2];
        sep |= (min3(p0, p1, p2) > r) | (max3(p0, p1, p2) < -r);
    }
    return sep;
}

struct ExpandArgs {
    const double* verts;
    const int32_t* tris;
    const uint32_t* parent_cells;
    const int32_t* pair_parent;
    const int32_t* pair_tri;
    int64_t npair;
    double cmin[3];
    double child_h;
};

// pass 1: hit byte per pair (bit o = octant o crossed), hit total per chunk
__global__ void __launch_bounds__(EXP_THREADS) expand_count_kernel(ExpandArgs a, uint8_t* hits,
                                                                   unsigned long long* chunk_sums) {
    __shared__ unsigned int s_total;
    if (threadIdx.x == 0) s_total = 0;
    __syncthreads();
    const int oct = threadIdx.x & 7;
    const double h = a.child_h * 0.5;
    const int64_t chunk0 = (int64_t)blockIdx.x * EXP_CHUNK;
    unsigned int mine = 0;
    for (int step = 0; step < EXP_CHUNK / 32; ++step) {
        const int64_t p = chunk0 + step * 32 + (threadIdx.x >> 3);
        bool hit = false;
        if (p < a.npair) {
            const int32_t t = a.pair_tri[p];
            const uint32_t* pc = a.parent_cells + 3 * (int64_t)a.pair_parent[p];
            const int32_t* tv = a.tris + 3 * (int64_t)t;
            const int64_t cc[3] = {(int64_t)pc[0] * 2 + (oct & 1), (int64_t)pc[1] * 2 + ((oct >> 1) & 1),
                                   (int64_t)pc[2] * 2 + ((oct >> 2) & 1)};
            double rel[3][3];
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {                          // KN:320-321
                const double centre = a.cmin[ax] + ((double)cc[ax] + 0.5) * a.child_h;
#pragma unroll
                for (int v = 0; v < 3; ++v) rel[ax][v] = a.verts[3 * (int64_t)tv[v] + ax] - centre;
            }
            hit = !sat_separated(rel[0], rel[1], rel[2], h);
        }
        const unsigned int b = __ballot_sync(0xffffffffu, hit);
        const int lane = threadIdx.x & 31;
        if ((lane & 7) == 0 && p < a.npair) hits[p] = (uint8_t)((b >> lane) & 0xffu);
        if (lane == 0) mine += __popc(b);
    }
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&s_total, mine);
    __syncthreads();
    if (threadIdx.x == 0) chunk_sums[blockIdx.x] = s_total;
}

// exclusive scan of n chunk totals in place by one block; the grand total goes to *total
__global__ void __launch_bounds__(1024) expand_scan_kernel(unsigned long long* sums, int64_t n,
                                                           unsigned long long* total) {
    __shared__ unsigned long long s_part[1024];
    const int64_t seg = (n + 1023) / 1024;
    const int64_t b = (int64_t)threadIdx.x * seg, e = b + seg < n ? b + seg : n;
    unsigned long long acc = 0;
    for (int64_t i = b; i < e; ++i) acc += sums[i];
    s_part[threadIdx.x] = acc;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {                       // Hillis-Steele, inclusive
        unsigned long long v = threadIdx.x >= off ? s_part[threadIdx.x - off] : 0;
        __syncthreads();
        s_part[threadIdx.x] += v;
        __syncthreads();
    }
    unsigned long long run = s_part[threadIdx.x] - acc;
    for (int64_t i = b; i < e; ++i) {
        const unsigned long long v = sums[i];
        sums[i] = run;
        run += v;
    }
    if (threadIdx.x == 1023) *total = s_part[1023];
}

// pass 2: thread order == output order, a ballot prefix gives the slot (np.nonzero order, KN:326)
__global__ void __launch_bounds__(EXP_THREADS) expand_emit_kernel(const uint32_t* parent_cells,
                                                                  const int32_t* pair_parent,
                                                                  const int32_t* pair_tri, int64_t npair,
                                                                  const uint8_t* hits,
                                                                  const unsigned long long* chunk_offs,
                                                                  uint32_t* out_cells, int32_t* out_tri) {
    __shared__ unsigned int s_warp[EXP_THREADS / 32];
    const int oct = threadIdx.x & 7, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t chunk0 = (int64_t)blockIdx.x * EXP_CHUNK;
    unsigned long long base = chunk_offs[blockIdx.x];
    for (int step = 0; step < EXP_CHUNK / 32; ++step) {
        const int64_t p = chunk0 + step * 32 + (threadIdx.x >> 3);
        const bool hit = p < npair && ((hits[p] >> oct) & 1);
        const unsigned int b = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) s_warp[warp] = __popc(b);
        __syncthreads();
        unsigned int before = 0, all = 0;
#pragma unroll
        for (int w = 0; w < EXP_THREADS / 32; ++w) {
            const unsigned int c = s_warp[w];
            before += w < warp ? c : 0;
            all += c;
        }
        if (hit) {
            const unsigned long long slot = base + before + __popc(b & ((1u << lane) - 1u));
            const uint32_t* pc = parent_cells + 3 * (int64_t)pair_parent[p];
            out_cells[3 * slot + 0] = pc[0] * 2u + (oct & 1);
            out_cells[3 * slot + 1] = pc[1] * 2u + ((oct >> 1) & 1);
            out_cells[3 * slot + 2] = pc[2] * 2u + ((oct >> 2) & 1);
            out_tri[slot] = pair_tri[p];
        }
        base += all;
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------------
// raycast

ML_DEV unsigned long long spread3(unsigned long long v) {
    v &= 0x1fffffULL;
    v = (v | (v << 32)) & 0x1f00000000ffffULL;
    v = (v | (v << 16)) & 0x1f0000ff0000ffULL;
    v = (v | (v << 8)) & 0x100f00f00f00f00fULL;
    v = (v | (v << 4)) & 0x10c30c30c30c30c3ULL;
    v = (v | (v << 2)) & 0x1249249249249249ULL;
    return v;
}
ML_DEV unsigned long long morton3(int64_t x, int64_t y, int64_t z) {
    return spread3((unsigned long long)x) | (spread3((unsigned long long)y) << 1) |
           (spread3((unsigned long long)z) << 2);
}

// np.searchsorted(keys, key) + the clamp / equality check of KN:453-455; -1 = not a leaf
ML_DEV int64_t find_key(const unsigned long long* __restrict__ keys, int64_t nkeys, unsigned long long key) {
    int64_t lo = 0, hi = nkeys;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(keys + mid) < key) lo = mid + 1; else hi = mid;
    }
    if (lo > nkeys - 1) lo = nkeys - 1;
    return (lo >= 0 && __ldg(keys + lo) == key) ? lo : -1;
}

// KN:335-358
ML_DEV double moller_trumbore(const double o[3], const double u[3], const double* __restrict__ v0,
                              const double* __restrict__ v1, const double* __restrict__ v2) {
    const double a0 = __ldg(v0), a1 = __ldg(v0 + 1), a2 = __ldg(v0 + 2);
    const double e1x = __ldg(v1) - a0, e1y = __ldg(v1 + 1) - a1, e1z = __ldg(v1 + 2) - a2;
    const double e2x = __ldg(v2) - a0, e2y = __ldg(v2 + 1) - a1, e2z = __ldg(v2 + 2) - a2;
    const double px = u[1] * e2z - u[2] * e2y;
    const double py = u[2] * e2x - u[0] * e2z;
    const double pz = u[0] * e2y - u[1] * e2x;
    const double det = (e1x * px + e1y * py) + e1z * pz;
    bool ok = det != 0.0;
    const double inv = __ddiv_rn(1.0, ok ? det : 1.0);
    const double tx = o[0] - a0, ty = o[1] - a1, tz = o[2] - a2;
    const double bu = ((tx * px + ty * py) + tz * pz) * inv;
    ok &= (bu >= 0.0) & (bu <= 1.0);
    const double qx = ty * e1z - tz * e1y;
    const double qy = tz * e1x - tx * e1z;
    const double qz = tx * e1y - ty * e1x;
    const double bv = ((u[0] * qx + u[1] * qy) + u[2] * qz) * inv;
    ok &= (bv >= 0.0) & (bu + bv <= 1.0);
    const double t = ((e2x * qx + e2y * qy) + e2z * qz) * inv;
    ok &= t >= 0.0;
    return ok ? t : INFINITY;
}

// astype(np.int64) + np.clip (KN:402-403, 511-512)
ML_DEV int64_t cell_of(double v, int64_t n_cells) {
    const int64_t c = (v != v || v < -9.0e18 || v > 9.0e18) ? INT64_MIN : (int64_t)v;
    return c < 0 ? 0 : (c > n_cells - 1 ? n_cells - 1 : c);
}

struct RayArgs {
    const double* origins;
    const double* dirs;
    int64_t nrays;
    const unsigned long long* keys;
    int64_t nkeys;
    const int64_t* offsets;
    const int32_t* tri_idx;
    const double* verts;
    const int32_t* tris;
    double cmin[3];
    double h;
    int64_t n_cells;
    const uint8_t* coarse;
    int64_t coarse_side;
    int coarse_shift;
    double* best_t;
    int32_t* best_tri;
    int64_t* leaf_pos;
};

__global__ void __launch_bounds__(128) raycast_kernel(RayArgs a) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.nrays) return;
    double o[3], u[3], inv_u[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) { o[k] = a.origins[3 * i + k]; u[k] = a.dirs[3 * i + k]; }
    double best_t = INFINITY;
    int32_t best_tri = -1;
    int64_t leaf = -1;
    double t_lo = 0.0, t_hi = INFINITY;
#pragma unroll
    for (int k = 0; k < 3; ++k) {                                    // KN:381-396 slab test
        const double cmax = a.cmin[k] + a.h * (double)a.n_cells;
        inv_u[k] = __ddiv_rn(1.0, u[k]);
        const bool ok_par = u[k] != 0.0;
        const double t1 = (a.cmin[k] - o[k]) * inv_u[k];
        const double t2 = (cmax - o[k]) * inv_u[k];
        if (ok_par) { t_lo = np_max(t_lo, np_min(t1, t2)); t_hi = np_min(t_hi, np_max(t1, t2)); }
        if (!ok_par && (o[k] < a.cmin[k] || o[k] > cmax)) t_hi = -INFINITY;
    }
    bool live = t_lo <= t_hi;
    if (live) {
        // n_cells <= 2^21 (checked by ml_raycast): 32-bit cell arithmetic in the march loop
        const int nc = (int)a.n_cells;
        const double t_start = np_max(t_lo, 0.0);
        int cell[3], step[3];
        double t_max[3], t_delta[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {                                // KN:400-416
            const double p = o[k] + t_start * u[k];
            cell[k] = (int)cell_of(__ddiv_rn(p - a.cmin[k], a.h), a.n_cells);
            step[k] = u[k] > 0.0 ? 1 : (u[k] < 0.0 ? -1 : 0);
            t_max[k] = INFINITY;
            t_delta[k] = INFINITY;
            if (u[k] != 0.0) {
                const double nxt = (double)(step[k] > 0 ? cell[k] + 1 : cell[k]);
                const double bound = a.cmin[k] + nxt * a.h;
                t_max[k] = (bound - o[k]) * inv_u[k];
                t_delta[k] = a.h * fabs(inv_u[k]);
            }
        }
        const int cs = a.coarse_shift;
        const unsigned int side = (unsigned int)a.coarse_side;
        double limit = np_min(best_t, t_hi);                         // min(best_t, t_hi) of KN:502
        const int64_t max_iter = 3 * a.n_cells + 3;
        for (int64_t it = 0; it < max_iter && live; ++it) {          // KN:420-503
            bool maybe = true;
            if (a.coarse)
                maybe = __ldg(a.coarse + ((size_t)((unsigned int)(cell[0] >> cs) * side +
                                                   (unsigned int)(cell[1] >> cs)) * side +
                                          (unsigned int)(cell[2] >> cs))) != 0;
            if (maybe) {
                const int64_t pos = find_key(a.keys, a.nkeys, morton3(cell[0], cell[1], cell[2]));
                if (pos >= 0) {
                    const int64_t jb = __ldg(a.offsets + pos), je = __ldg(a.offsets + pos + 1);
                    for (int64_t j = jb; j < je; ++j) {
                        const int32_t f = __ldg(a.tri_idx + j);
                        const int32_t* tv = a.tris + 3 * (int64_t)f;
                        const double t = moller_trumbore(o, u, a.verts + 3 * (int64_t)__ldg(tv),
                                                         a.verts + 3 * (int64_t)__ldg(tv + 1),
                                                         a.verts + 3 * (int64_t)__ldg(tv + 2));
                        if (t < best_t || (t == best_t && f < best_tri)) {   // KN:470-487
                            best_t = t;
                            best_tri = f;
                            limit = np_min(best_t, t_hi);
                        }
                    }
                }
            }
            // KN:490-503; dynamic register-array indexing would spill: select by hand
            double cur;
            int c;
            if (t_max[0] <= t_max[1] && t_max[0] <= t_max[2]) {
                cur = t_max[0]; cell[0] += step[0]; t_max[0] += t_delta[0]; c = cell[0];
            } else if (t_max[1] <= t_max[2]) {
                cur = t_max[1]; cell[1] += step[1]; t_max[1] += t_delta[1]; c = cell[1];
            } else {
                cur = t_max[2]; cell[2] += step[2]; t_max[2] += t_delta[2]; c = cell[2];
            }
            if ((unsigned int)c >= (unsigned int)nc || cur > limit) live = false;
        }
        if (isfinite(best_t) && best_tri >= 0) {                     // KN:506-524
            int64_t lc[3];
#pragma unroll
            for (int k = 0; k < 3; ++k)
                lc[k] = cell_of(__ddiv_rn((o[k] + best_t * u[k]) - a.cmin[k], a.h), a.n_cells);
            leaf = find_key(a.keys, a.nkeys, morton3(lc[0], lc[1], lc[2]));
            if (leaf < 0) { best_t = INFINITY; best_tri = -1; }
        }
    }
    a.best_t[i] = best_t;
    a.best_tri[i] = best_tri;
    a.leaf_pos[i] = leaf;
}

// ---------------------------------------------------------------------------------------------
// ray set-up of an octree edit (one ray per window pixel inside the tool shape)

struct ToolRayArgs {
    double inv[16];                 // inverse view-projection, row major
    double left, bottom;            // window position of the tool bitmap's lower-left corner
    int x0, y0, nx, ny;             // pixel box of the tool in the window
    int cam_w, cam_h, tw, th;
    const uint8_t* shape;
    double* origins;
    double* dirs;
    unsigned long long* count;
};

// One thread per pixel of the tool's box.  A pixel whose centre maps into a set texel of the tool bitmap
// (the tool map of KN:187-192, half open at the far edges) gets the ray through its centre: origin on the
// near plane, unit direction.  Every other pixel gets a NaN direction, which ml_raycast reports as a miss
// after the slab test -- so the edit needs no stream compaction.
__global__ void __launch_bounds__(256) tool_rays_kernel(ToolRayArgs a) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = a.nx * a.ny;
    bool keep = false;
    if (i < n) {
        const int iy = i / a.nx, ix = i - iy * a.nx;
        const double gx = (double)(a.x0 + ix) + 0.5, gy = (double)(a.y0 + iy) + 0.5;
        const double s = (gx - a.left) / (double)a.tw, t = (gy - a.bottom) / (double)a.th;
        if (s >= 0.0 && s < 1.0 && t >= 0.0 && t < 1.0) {
            int si = (int)(s * (double)a.tw), ti = (int)(t * (double)a.th);
            si = si > a.tw - 1 ? a.tw - 1 : si;
            ti = ti > a.th - 1 ? a.th - 1 : ti;
            keep = a.shape[(size_t)ti * a.tw + si] != 0;
        }
        double o[3] = {0.0, 0.0, 0.0}, d[3] = {NAN, NAN, NAN};
        if (keep) {
            const double vx = gx / (double)a.cam_w * 2.0 - 1.0, vy = gy / (double)a.cam_h * 2.0 - 1.0;
            double pn[4], pf[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const double base = (a.inv[4 * r] * vx + a.inv[4 * r + 1] * vy) + a.inv[4 * r + 3];
                pn[r] = base - a.inv[4 * r + 2];
                pf[r] = base + a.inv[4 * r + 2];
            }
            double len2 = 0.0;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                o[k] = pn[k] / pn[3];
                d[k] = pf[k] / pf[3] - o[k];
                len2 += d[k] * d[k];
            }
            const double len = sqrt(len2);
#pragma unroll
            for (int k = 0; k < 3; ++k) d[k] /= len;
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) { a.origins[3 * (size_t)i + k] = o[k]; a.dirs[3 * (size_t)i + k] = d[k]; }
    }
    const unsigned int b = __ballot_sync(0xffffffffu, keep);
    if ((threadIdx.x & 31) == 0 && b && a.count) atomicAdd(a.count, (unsigned long long)__popc(b));
}

inline int64_t chunks_of(int64_t npair) { return (npair + EXP_CHUNK - 1) / EXP_CHUNK; }

}  // namespace

extern "C" {

size_t ml_expand_pairs_workspace_bytes(int64_t npair) {
    if (npair < 0) npair = 0;
    const size_t hits = ((size_t)npair + 255) & ~(size_t)255;
    return hits + (size_t)(chunks_of(npair) + 1) * sizeof(unsigned long long);
}

int ml_expand_pairs_count(const double* verts, const int32_t* tris, const uint32_t* parent_cells,
                          const int32_t* pair_parent, const int32_t* pair_tri, int64_t npair,
                          const double* cube_min, double child_h, void* workspace, size_t workspace_bytes,
                          uint64_t* total, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (npair < 0 || !total || !cube_min) return ml_fail(ML_ERR_ARG, "ml_expand_pairs_count: bad arguments");
    if (npair == 0) {                                                // KN:307-309
        ML_CUDA(cudaMemsetAsync(total, 0, sizeof(uint64_t), st));
        return ML_OK;
    }
    if (!verts || !tris || !parent_cells || !pair_parent || !pair_tri || !workspace ||
        workspace_bytes < ml_expand_pairs_workspace_bytes(npair))
        return ml_fail(ML_ERR_ARG, "ml_expand_pairs_count: null input or workspace too small");
    ExpandArgs a;
    a.verts = verts; a.tris = tris; a.parent_cells = parent_cells; a.pair_parent = pair_parent;
    a.pair_tri = pair_tri; a.npair = npair; a.child_h = child_h;
    for (int k = 0; k < 3; ++k) a.cmin[k] = cube_min[k];
    uint8_t* hits = (uint8_t*)workspace;
    unsigned long long* sums = (unsigned long long*)(hits + (((size_t)npair + 255) & ~(size_t)255));
    const int64_t nchunk = chunks_of(npair);
    expand_count_kernel<<<(unsigned)nchunk, EXP_THREADS, 0, st>>>(a, hits, sums);
    expand_scan_kernel<<<1, 1024, 0, st>>>(sums, nchunk, (unsigned long long*)total);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int ml_expand_pairs_emit(const uint32_t* parent_cells, const int32_t* pair_parent, const int32_t* pair_tri,
                         int64_t npair, const void* workspace, uint32_t* out_cells, int32_t* out_tri,
                         void* stream) {
    if (npair < 0) return ml_fail(ML_ERR_ARG, "ml_expand_pairs_emit: bad arguments");
    if (npair == 0) return ML_OK;
    if (!parent_cells || !pair_parent || !pair_tri || !workspace || !out_cells || !out_tri)
        return ml_fail(ML_ERR_ARG, "ml_expand_pairs_emit: null pointer");
    const uint8_t* hits = (const uint8_t*)workspace;
    const unsigned long long* offs =
        (const unsigned long long*)(hits + (((size_t)npair + 255) & ~(size_t)255));
    expand_emit_kernel<<<(unsigned)chunks_of(npair), EXP_THREADS, 0, (cudaStream_t)stream>>>(
        parent_cells, pair_parent, pair_tri, npair, hits, offs, out_cells, out_tri);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int ml_raycast(const double* origins, const double* dirs, int64_t nrays, const uint64_t* keys, int64_t nkeys,
               const int64_t* offsets, const int32_t* tri_idx, const double* verts, const int32_t* tris,
               const double* cube_min, double h, int64_t n_cells, const uint8_t* coarse, int64_t coarse_side,
               int coarse_shift, double* best_t, int32_t* best_tri, int64_t* leaf_pos, void* stream) {
    if (nrays < 0 || nkeys < 0 || n_cells < 1 || n_cells > (1 << 21) || !cube_min ||
        (coarse && (coarse_side < 1 || coarse_shift < 0 || coarse_shift > 21 ||
                    ((n_cells - 1) >> coarse_shift) >= coarse_side)))
        return ml_fail(ML_ERR_ARG, "ml_raycast: bad arguments (n_cells <= 2^21, coarse map must cover the grid)");
    if (nrays == 0) return ML_OK;
    if (!origins || !dirs || !best_t || !best_tri || !leaf_pos ||
        (nkeys > 0 && (!keys || !offsets || !tri_idx || !verts || !tris)))
        return ml_fail(ML_ERR_ARG, "ml_raycast: null pointer");
    RayArgs a;
    a.origins = origins; a.dirs = dirs; a.nrays = nrays;
    a.keys = (const unsigned long long*)keys; a.nkeys = nkeys; a.offsets = offsets; a.tri_idx = tri_idx;
    a.verts = verts; a.tris = tris; a.h = h; a.n_cells = n_cells;
    for (int k = 0; k < 3; ++k) a.cmin[k] = cube_min[k];
    a.coarse = coarse; a.coarse_side = coarse_side; a.coarse_shift = coarse_shift;
    a.best_t = best_t; a.best_tri = best_tri; a.leaf_pos = leaf_pos;
    raycast_kernel<<<(unsigned)((nrays + 63) / 64), 64, 0, (cudaStream_t)stream>>>(a);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int ml_tool_rays(const double* inv_view_proj, int64_t cam_w, int64_t cam_h, double tool_px, double tool_py,
                 const uint8_t* shape, int64_t shape_w, int64_t shape_h, int64_t x0, int64_t y0, int64_t nx, int64_t ny,
                 double* origins, double* dirs, uint64_t* count, void* stream) {
    if (!inv_view_proj || cam_w < 1 || cam_h < 1 || shape_w < 1 || shape_h < 1 || nx < 0 || ny < 0 ||
        nx * ny > (int64_t)1 << 30)
        return ml_fail(ML_ERR_ARG, "ml_tool_rays: bad arguments");
    if (nx == 0 || ny == 0) return ML_OK;
    if (!shape || !origins || !dirs) return ml_fail(ML_ERR_ARG, "ml_tool_rays: null pointer");
    ToolRayArgs a;
    for (int k = 0; k < 16; ++k) a.inv[k] = inv_view_proj[k];
    a.left = tool_px - 0.5 * (double)shape_w;
    a.bottom = tool_py - 0.5 * (double)shape_h;
    a.x0 = (int)x0; a.y0 = (int)y0; a.nx = (int)nx; a.ny = (int)ny;
    a.cam_w = (int)cam_w; a.cam_h = (int)cam_h; a.tw = (int)shape_w; a.th = (int)shape_h;
    a.shape = shape; a.origins = origins; a.dirs = dirs; a.count = (unsigned long long*)count;
    tool_rays_kernel<<<(unsigned)((nx * ny + 255) / 256), 256, 0, (cudaStream_t)stream>>>(a);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

}  // extern "C"
