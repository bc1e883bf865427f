// Layer algebra (north star (3)): union / intersection / difference / masking over (data, mask)
// layers.  The reference leaves inter-layer algebra out of scope; the frozen
// definition is oracle/kn_port.c ext_layer_op.
//
// Pure HBM streams.  One thread step covers 16 texels: a 128-bit load of each mask plane and
// ESIZE 128-bit loads of each data plane, all issued before the first use, then SIMD-in-register
// byte logic and 128-bit stores.  Algorithmic traffic per texel: mask-only 3 B (2 reads + 1
// write), full layers 3*(1+ESIZE) B, N-layer fused chain (N+1)*(1+ESIZE) B.
#include "common.cuh"
#include "meshlayers_b200.h"
#include "internal.h"

namespace {

constexpr int BLOCK = 256;
constexpr int MAX_CHAIN = 16;

// 0xff in every byte lane of m that is non-zero
ML_DEV uint32_t nz_bytes(uint32_t m) { return __vcmpne4(m, 0u); }

// expand the 4 byte-lane flags of `ff` (each 0x00 / 0xff) to element lanes of ESIZE bytes:
// word j (0 <= j < ESIZE) of the 4-element group
template <int ESIZE> ML_DEV uint32_t expand(uint32_t ff, int j);
template <> ML_DEV uint32_t expand<1>(uint32_t ff, int) { return ff; }
template <> ML_DEV uint32_t expand<2>(uint32_t ff, int j) { return __byte_perm(ff, 0u, j == 0 ? 0x1100 : 0x3322); }
template <> ML_DEV uint32_t expand<4>(uint32_t ff, int j) {
    return __byte_perm(ff, 0u, j == 0 ? 0x0000 : j == 1 ? 0x1111 : j == 2 ? 0x2222 : 0x3333);
}

// One 4-texel group: masks as byte flags (ff), data words d[ESIZE].
template <int ESIZE>
struct Group {
    uint32_t ff;                 // 0xff per valid texel
    uint32_t d[ESIZE > 0 ? ESIZE : 1];
};

template <int ESIZE>
ML_DEV void combine(int op, Group<ESIZE>& acc, const Group<ESIZE>& b) {
    uint32_t keep_a, take_b, out_ff;
    switch (op) {
    case ML_OP_UNION:        out_ff = acc.ff | b.ff;  keep_a = acc.ff;  take_b = b.ff & ~acc.ff; break;
    case ML_OP_DIFFERENCE:   out_ff = acc.ff & ~b.ff; keep_a = out_ff;  take_b = 0u; break;
    default:                 out_ff = acc.ff & b.ff;  keep_a = out_ff;  take_b = 0u; break;   // intersection / masking
    }
    if (ESIZE > 0) {
#pragma unroll
        for (int j = 0; j < (ESIZE > 0 ? ESIZE : 1); ++j)
            acc.d[j] = (acc.d[j] & expand<(ESIZE > 0 ? ESIZE : 1)>(keep_a, j)) |
                       (b.d[j] & expand<(ESIZE > 0 ? ESIZE : 1)>(take_b, j));
    }
    acc.ff = out_ff;
}

struct ChainArgs {
    const void* data[MAX_CHAIN];
    const uint8_t* mask[MAX_CHAIN];
    int ops[MAX_CHAIN];
    int nlayers;
};

// 16 texels per thread step.  Layers are fetched in groups of GL (all GL*(1+ESIZE) 128-bit
// requests of a group are issued before the first use), then folded into the accumulator left
// to right.  GL is chosen so a group fits the register file: 8 / 8 / 4 / 2 for ESIZE 0/1/2/4.
template <int ESIZE> struct GroupLen { static constexpr int value = ESIZE <= 1 ? 8 : (ESIZE == 2 ? 4 : 2); };

template <int ESIZE>
__global__ void __launch_bounds__(BLOCK)
chain_kernel(ChainArgs a, void* dc, uint8_t* mc, long long n) {
    constexpr int ES = ESIZE > 0 ? ESIZE : 1;
    constexpr int GL = GroupLen<ESIZE>::value;
    const long long tid = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * BLOCK;
    const long long nv = n >> 4;
    const bool eager = (a.ops[0] & ML_CHAIN_EAGER) != 0;
    for (long long v = tid; v < nv; v += nthreads) {
        Group<ESIZE> acc[4];                      // four 4-texel groups of the 16-texel vector
        for (int l0 = 0; l0 < a.nlayers; l0 += GL) {
            uint4 m[GL];
            uint4 d[GL][ES];
#pragma unroll
            for (int k = 0; k < GL; ++k) {
                if (l0 + k < a.nlayers) {
                    m[k] = ld_stream_rw((const uint4*)a.mask[l0 + k] + v);
                    if (ESIZE > 0) {
                        // only the first operand and union operands can supply a data value (combine():
                        // take_b); the data planes of the other operands are not read unless ML_CHAIN_EAGER
                        const bool need = eager || l0 + k == 0 || a.ops[l0 + k] == ML_OP_UNION;
#pragma unroll
                        for (int j = 0; j < ES; ++j)
                            d[k][j] = need ? ld_stream_rw((const uint4*)a.data[l0 + k] + v * ES + j) : make_uint4(0u, 0u, 0u, 0u);
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < GL; ++k) {
                if (l0 + k < a.nlayers) {
                    const int op = a.ops[l0 + k];
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        Group<ESIZE> b;
                        b.ff = nz_bytes(((const uint32_t*)&m[k])[g]);
                        if (ESIZE > 0) {
#pragma unroll
                            for (int j = 0; j < ES; ++j) b.d[j] = ((const uint32_t*)&d[k][0])[g * ES + j];
                        }
                        if (l0 + k == 0) {        // first operand initialises the accumulator
                            acc[g].ff = b.ff;
                            if (ESIZE > 0) {
#pragma unroll
                                for (int j = 0; j < ES; ++j) acc[g].d[j] = b.d[j] & expand<ES>(b.ff, j);
                            }
                        } else {
                            combine<ESIZE>(op, acc[g], b);
                        }
                    }
                }
            }
        }
        uint4 om;
        uint4 od[ES];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            ((uint32_t*)&om)[g] = acc[g].ff & 0x01010101u;
            if (ESIZE > 0) {
#pragma unroll
                for (int j = 0; j < ES; ++j) ((uint32_t*)&od[0])[g * ES + j] = acc[g].d[j];
            }
        }
        st_stream((uint4*)mc + v, om);
        if (ESIZE > 0) {
#pragma unroll
            for (int j = 0; j < ES; ++j) st_stream((uint4*)dc + v * ES + j, od[j]);
        }
    }
    // tail (< 16 texels) and nothing else: scalar
    for (long long i = (nv << 4) + tid; i < n; i += nthreads) {
        bool am = a.mask[0][i] != 0;
        uint32_t ad = 0;
        if (ESIZE == 1) ad = ((const uint8_t*)a.data[0])[i];
        if (ESIZE == 2) ad = ((const uint16_t*)a.data[0])[i];
        if (ESIZE == 4) ad = ((const uint32_t*)a.data[0])[i];
        if (!am) ad = 0;
        for (int l = 1; l < a.nlayers; ++l) {
            const bool bm = a.mask[l][i] != 0;
            uint32_t bd = 0;
            if (ESIZE == 1) bd = ((const uint8_t*)a.data[l])[i];
            if (ESIZE == 2) bd = ((const uint16_t*)a.data[l])[i];
            if (ESIZE == 4) bd = ((const uint32_t*)a.data[l])[i];
            switch (a.ops[l]) {
            case ML_OP_UNION:      if (!am && bm) ad = bd; am = am || bm; break;
            case ML_OP_DIFFERENCE: am = am && !bm; if (!am) ad = 0; break;
            default:               am = am && bm;  if (!am) ad = 0; break;
            }
        }
        mc[i] = am ? 1 : 0;
        if (ESIZE == 1) ((uint8_t*)dc)[i] = (uint8_t)ad;
        if (ESIZE == 2) ((uint16_t*)dc)[i] = (uint16_t)ad;
        if (ESIZE == 4) ((uint32_t*)dc)[i] = ad;
    }
}

// Chains of 3 to 8 layers with data (label layers of 1, 2 or 4 bytes) read their data planes LAZILY.
// The masks alone decide which layers can contribute a data value to a 16-texel vector: the first
// operand where its mask is set, a union operand where it fills texels the accumulator does not hold
// yet; intersection / difference / masking operands never do.  A dry run of the mask fold finds
// them and only their data vectors are fetched -- thematic layers are sparse, so most data vectors
// are never read (8 masks + 2 output bytes per texel instead of 18).  The mask -> data dependency is
// hidden by software pipelining: the masks of the thread's NEXT vector are requested before the data
// of the current one, so as many bytes are in flight as in the eager kernel.  Per vector: (1) dry run of the mask
// fold -> final mask + the set of layers that matter; (2) their data vectors are requested; (3) while they are in
// flight a second masks-only pass records, per texel, WHICH operand supplied its value (one-hot source byte);
// (4) the data vectors are gathered by source; (5) the final mask clears what was removed.
#ifndef ML_CHAIN_LAZY_MINB
#define ML_CHAIN_LAZY_MINB 2
#endif

template <int ESIZE>
__global__ void __launch_bounds__(BLOCK, ML_CHAIN_LAZY_MINB)
chain_lazy_kernel(ChainArgs a, void* dc, uint8_t* mc, long long nv) {
    constexpr int GL = 8;
    const long long tid = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * BLOCK;
    // ma: the vector being folded; mb: the next vector's masks, requested before the current vector's data
    uint4 ma[GL], mb[GL];
    if (tid < nv) {
#pragma unroll
        for (int k = 0; k < GL; ++k) if (k < a.nlayers) ma[k] = ld_stream_rw((const uint4*)a.mask[k] + tid);
    }
    auto step = [&](const long long v, uint4 (&m)[GL], uint4 (&mn)[GL]) {
        if (v + nthreads < nv) {
#pragma unroll
            for (int k = 0; k < GL; ++k) if (k < a.nlayers) mn[k] = ld_stream_rw((const uint4*)a.mask[k] + v + nthreads);
        }
        // The fold works on mask bytes that are exactly 0 / 1 (what every writer of this library stores); a vector
        // holding any other non-zero byte value is normalised first (rare: caller-made planes).
        uint32_t odd = 0u;
#pragma unroll
        for (int k = 0; k < GL; ++k)
            if (k < a.nlayers) odd |= (m[k].x | m[k].y | m[k].z | m[k].w) & 0xfefefefeu;
        if (odd) {
#pragma unroll
            for (int k = 0; k < GL; ++k) {
                if (k < a.nlayers) {
#pragma unroll
                    for (int g = 0; g < 4; ++g) ((uint32_t*)&m[k])[g] = nz_bytes(((const uint32_t*)&m[k])[g]) & 0x01010101u;
                }
            }
        }
        // Pass 1 -- the mask fold alone, in the 0 / 1 byte domain (one or two LOP3 per word and layer): final mask
        // `sim`, and which layers' data can reach the result of this vector (the first operand where its mask is set,
        // a union operand where it fills texels the accumulator does not hold; intersection / difference / masking
        // operands never).
        unsigned need = 0;
        uint32_t sim[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int k = 0; k < GL; ++k) {
            if (k < a.nlayers) {
                const int op = a.ops[k];
                uint32_t fills = 0u;
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const uint32_t bm = ((const uint32_t*)&m[k])[g];
                    if (k == 0) { fills |= bm; sim[g] = bm; }
                    else if (op == ML_OP_UNION) { fills |= bm & ~sim[g]; sim[g] |= bm; }
                    else if (op == ML_OP_DIFFERENCE) sim[g] &= ~bm;
                    else sim[g] &= bm;
                }
                if (fills) need |= 1u << k;
            }
        }
        const uint4 om = make_uint4(sim[0], sim[1], sim[2], sim[3]);
        uint4 od[ESIZE];
        // warp-uniform choice: a warp that took both branches would pay for both (dense / mixed layers)
        if (__all_sync(__activemask(), need <= 1u)) {
            // no union operand fills anything: the result's data is the first operand's under the final mask
            // (need == 1), or nothing at all (need == 0: the first operand is empty here and so is the result)
#pragma unroll
            for (int j = 0; j < ESIZE; ++j) od[j] = make_uint4(0u, 0u, 0u, 0u);
            if (need) {
#pragma unroll
                for (int j = 0; j < ESIZE; ++j) {
                    const uint4 d0 = ld_stream_rw((const uint4*)a.data[0] + v * ESIZE + j);
                    od[j] = d0;
                }
#pragma unroll
                for (int g = 0; g < 4; ++g)
#pragma unroll
                    for (int j = 0; j < ESIZE; ++j)
                        ((uint32_t*)&od[0])[g * ESIZE + j] &= expand<ESIZE>(sim[g] * 0xffu, j);
            }
        } else {
            // one-byte layers: all needed vectors are requested together; wider layers (64 bytes per
            // layer and vector) are fetched one layer at a time inside the fold to bound the registers
            uint4 d1[ESIZE == 1 ? GL : 1];                  // d1[k] is defined (and read) only where bit k of `need` is set
            if (ESIZE == 1) {
                long long off = v << 4;                     // one byte offset for all planes (opaque: no per-plane re-derivation)
                asm volatile("" : "+l"(off));
#pragma unroll
                for (int k = 0; k < GL; ++k)
                    if ((need >> k) & 1u) d1[k] = ld_stream_rw((const uint4*)((const uint8_t*)a.data[k] + off));
            }
            // Pass 2a -- masks only, so it runs while the data vectors requested above are in flight: a one-hot SOURCE
            // byte per texel, bit k set where union operand k (or the first operand, bit 0) supplied a value, i.e. filled
            // a texel the accumulator did not hold at that point.  Bits are only ever added: a texel that is removed and
            // filled again later carries two bits and the gather below lets the later layer win; a removed texel that
            // never comes back is cleared by the final mask.
            uint32_t cur[4] = {0u, 0u, 0u, 0u};             // the accumulator's mask (0 / 1 bytes) while folding
            uint32_t src[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int k = 0; k < GL; ++k) {
                if (k < a.nlayers) {
                    const int op = a.ops[k];
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        const uint32_t bm = ((const uint32_t*)&m[k])[g];
                        if (k == 0) { cur[g] = bm; src[g] = bm; }
                        else if (op == ML_OP_UNION) { src[g] += (bm & ~cur[g]) << k; cur[g] |= bm; }    // bit k is new: + is |
                        else if (op == ML_OP_DIFFERENCE) cur[g] &= ~bm;
                        else cur[g] &= bm;
                    }
                }
            }
            // Pass 2b -- the gather, in layer order (a later source overwrites an earlier one), restricted to the layers
            // some lane of the warp needs (warp-uniform branch: a per-lane predicate would still issue the instructions)
            const unsigned wneed = __reduce_or_sync(__activemask(), need);
            uint32_t accd[4 * ESIZE];
#pragma unroll
            for (int i = 0; i < 4 * ESIZE; ++i) accd[i] = 0u;
#pragma unroll
            for (int k = 0; k < GL; ++k) {
                if (k < a.nlayers && ((wneed >> k) & 1u)) {
                    const bool needed = (need >> k) & 1u;
                    uint4 dk[ESIZE];
                    if (ESIZE == 1) dk[0] = d1[k];         // plain alias: read only under `needed`, where it is defined
                    else if (needed) {
#pragma unroll
                        for (int j = 0; j < ESIZE; ++j) dk[j] = ld_stream_rw((const uint4*)a.data[k] + v * ESIZE + j);
                    }
                    if (needed) {
#pragma unroll
                        for (int g = 0; g < 4; ++g) {
                            const uint32_t take = ((src[g] >> k) & 0x01010101u) * 0xffu;
#pragma unroll
                            for (int j = 0; j < ESIZE; ++j) {
                                const uint32_t t = expand<ESIZE>(take, j);
                                accd[g * ESIZE + j] = (accd[g * ESIZE + j] & ~t) | (((const uint32_t*)&dk[0])[g * ESIZE + j] & t);
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int g = 0; g < 4; ++g)
#pragma unroll
                for (int j = 0; j < ESIZE; ++j) ((uint32_t*)&od[0])[g * ESIZE + j] = accd[g * ESIZE + j] & expand<ESIZE>(sim[g] * 0xffu, j);
        }
        st_stream((uint4*)mc + v, om);
#pragma unroll
        for (int j = 0; j < ESIZE; ++j) st_stream((uint4*)dc + v * ESIZE + j, od[j]);
    };
    for (long long v = tid; v < nv; v += nthreads) {
        step(v, ma, mb);
#pragma unroll
        for (int k = 0; k < GL; ++k) ma[k] = mb[k];     // (unrolling by two with the buffers swapped spills: 0.54 -> 0.72 ms)
    }
}

// fully scalar kernel for planes that are not 16-byte aligned
template <int ESIZE>
__global__ void __launch_bounds__(BLOCK)
chain_scalar_kernel(ChainArgs a, void* dc, uint8_t* mc, long long n) {
    const long long nthreads = (long long)gridDim.x * BLOCK;
    for (long long i = (long long)blockIdx.x * BLOCK + threadIdx.x; i < n; i += nthreads) {
        bool am = a.mask[0][i] != 0;
        uint32_t ad = 0;
        if (ESIZE == 1) ad = ((const uint8_t*)a.data[0])[i];
        if (ESIZE == 2) ad = ((const uint16_t*)a.data[0])[i];
        if (ESIZE == 4) ad = ((const uint32_t*)a.data[0])[i];
        if (!am) ad = 0;
        for (int l = 1; l < a.nlayers; ++l) {
            const bool bm = a.mask[l][i] != 0;
            uint32_t bd = 0;
            if (ESIZE == 1) bd = ((const uint8_t*)a.data[l])[i];
            if (ESIZE == 2) bd = ((const uint16_t*)a.data[l])[i];
            if (ESIZE == 4) bd = ((const uint32_t*)a.data[l])[i];
            switch (a.ops[l]) {
            case ML_OP_UNION:      if (!am && bm) ad = bd; am = am || bm; break;
            case ML_OP_DIFFERENCE: am = am && !bm; if (!am) ad = 0; break;
            default:               am = am && bm;  if (!am) ad = 0; break;
            }
        }
        mc[i] = am ? 1 : 0;
        if (ESIZE == 1) ((uint8_t*)dc)[i] = (uint8_t)ad;
        if (ESIZE == 2) ((uint16_t*)dc)[i] = (uint16_t)ad;
        if (ESIZE == 4) ((uint32_t*)dc)[i] = ad;
    }
}

// Binary operator fast path (the 3 B/texel kernel): VPT 16-texel vectors per thread step, ALL
// operand loads of the step issued before the first store (the chain kernel cannot hoist loads
// over its stores because its output may alias an input), so each thread keeps
// VPT*2*(1+ESIZE) 128-bit requests in flight.  A thread only ever reads the vectors it writes,
// so in-place use (output aliasing A) stays race-free.
template <int ESIZE, int VPT>
__global__ void __launch_bounds__(BLOCK)
binary_kernel(ChainArgs a, void* dc, uint8_t* mc, long long nv) {
    constexpr int ES = ESIZE > 0 ? ESIZE : 1;
    const long long tid = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * BLOCK;
    const int op = a.ops[1];
    const bool need_b = op == ML_OP_UNION;     // only a union can take a data value from B (combine(): take_b)
    for (long long v0 = tid; v0 < nv; v0 += nthreads * VPT) {
        uint4 m[VPT][2];
        uint4 d[VPT][2][ES];
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            const long long v = v0 + k * nthreads;
            if (v < nv) {
#pragma unroll
                for (int l = 0; l < 2; ++l) {
                    m[k][l] = ld_stream_rw((const uint4*)a.mask[l] + v);
                    if (ESIZE > 0) {
#pragma unroll
                        for (int j = 0; j < ES; ++j)
                            d[k][l][j] = (l == 0 || need_b) ? ld_stream_rw((const uint4*)a.data[l] + v * ES + j)
                                                            : make_uint4(0u, 0u, 0u, 0u);
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            const long long v = v0 + k * nthreads;
            if (v >= nv) break;
            uint4 om;
            uint4 od[ES];
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                Group<ESIZE> acc, b;
                acc.ff = nz_bytes(((const uint32_t*)&m[k][0])[g]);
                b.ff = nz_bytes(((const uint32_t*)&m[k][1])[g]);
                if (ESIZE > 0) {
#pragma unroll
                    for (int j = 0; j < ES; ++j) {
                        acc.d[j] = ((const uint32_t*)&d[k][0][0])[g * ES + j] & expand<ES>(acc.ff, j);
                        b.d[j] = ((const uint32_t*)&d[k][1][0])[g * ES + j];
                    }
                }
                combine<ESIZE>(op, acc, b);
                ((uint32_t*)&om)[g] = acc.ff & 0x01010101u;
                if (ESIZE > 0) {
#pragma unroll
                    for (int j = 0; j < ES; ++j) ((uint32_t*)&od[0])[g * ES + j] = acc.d[j];
                }
            }
            st_stream((uint4*)mc + v, om);
            if (ESIZE > 0) {
#pragma unroll
                for (int j = 0; j < ES; ++j) st_stream((uint4*)dc + v * ES + j, od[j]);
            }
        }
    }
}

inline bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

template <int ESIZE>
int launch_chain(const ChainArgs& a, void* dc, uint8_t* mc, long long n, cudaStream_t st) {
    bool vec = aligned16(mc) && (ESIZE == 0 || aligned16(dc));
    for (int l = 0; l < a.nlayers; ++l) vec = vec && aligned16(a.mask[l]) && (ESIZE == 0 || aligned16(a.data[l]));
    if (vec && a.nlayers == 2 && ESIZE <= 2 && (n >> 4) > 0) {
        constexpr int VPT = ESIZE == 0 ? 4 : 2;
        const long long nv = n >> 4;
        long long blocks = (nv + (long long)BLOCK * VPT - 1) / ((long long)BLOCK * VPT);
        const long long cap = (long long)ml_sm_count() * 8;
        if (blocks > cap) blocks = cap;
        binary_kernel<ESIZE, VPT><<<(unsigned)blocks, BLOCK, 0, st>>>(a, dc, mc, nv);
        ML_CUDA(cudaGetLastError());
        const long long tail = n & 15;
        if (tail == 0) return ML_OK;
        // the last < 16 texels go through the scalar kernel on shifted pointers
        ChainArgs t = a;
        const long long off = nv << 4;
        for (int l = 0; l < 2; ++l) {
            t.mask[l] = a.mask[l] + off;
            if (ESIZE > 0) t.data[l] = (const uint8_t*)a.data[l] + off * ESIZE;
        }
        chain_scalar_kernel<ESIZE><<<1, BLOCK, 0, st>>>(t, ESIZE > 0 ? (void*)((uint8_t*)dc + off * ESIZE) : nullptr, mc + off, tail);
        ML_CUDA(cudaGetLastError());
        return ML_OK;
    }
    if (vec && ESIZE >= 1 && a.nlayers > 2 && a.nlayers <= 8 && (n >> 4) > 0 && !(a.ops[0] & ML_CHAIN_EAGER)) {
        const long long nv = n >> 4;
        long long blocks = (nv + BLOCK - 1) / BLOCK;
        const long long cap = (long long)ml_sm_count() * 16;
        if (blocks > cap) blocks = cap;
        chain_lazy_kernel<(ESIZE > 0 ? ESIZE : 1)><<<(unsigned)blocks, BLOCK, 0, st>>>(a, dc, mc, nv);
        ML_CUDA(cudaGetLastError());
        const long long tail = n & 15;
        if (tail == 0) return ML_OK;
        ChainArgs t = a;
        const long long off = nv << 4;
        for (int l = 0; l < a.nlayers; ++l) { t.mask[l] = a.mask[l] + off; t.data[l] = (const uint8_t*)a.data[l] + off * ESIZE; }
        chain_scalar_kernel<ESIZE><<<1, BLOCK, 0, st>>>(t, (void*)((uint8_t*)dc + off * ESIZE), mc + off, tail);
        ML_CUDA(cudaGetLastError());
        return ML_OK;
    }
    const long long items = vec ? ((n + 15) >> 4) : n;
    long long blocks = (items + BLOCK - 1) / BLOCK;
    const long long cap = (long long)ml_sm_count() * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    if (vec) chain_kernel<ESIZE><<<(unsigned)blocks, BLOCK, 0, st>>>(a, dc, mc, n);
    else chain_scalar_kernel<ESIZE><<<(unsigned)blocks, BLOCK, 0, st>>>(a, dc, mc, n);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

int dispatch_chain(const ChainArgs& a, void* dc, uint8_t* mc, int esize, long long n, cudaStream_t st) {
    if (n <= 0) return ML_OK;
    switch (esize) {
    case 0: return launch_chain<0>(a, dc, mc, n, st);
    case 1: return launch_chain<1>(a, dc, mc, n, st);
    case 2: return launch_chain<2>(a, dc, mc, n, st);
    case 4: return launch_chain<4>(a, dc, mc, n, st);
    }
    return ml_fail(ML_ERR_ARG, "esize must be 0 (mask only), 1, 2 or 4");
}

}  // namespace

extern "C" {

int ml_layer_op(int op, const void* da, const uint8_t* ma, const void* db, const uint8_t* mb,
                void* dc, uint8_t* mc, int esize, int64_t n, void* stream) {
    if (op < ML_OP_UNION || op > ML_OP_MASKING) return ml_fail(ML_ERR_ARG, "unknown layer operator");
    ChainArgs a;
    a.nlayers = 2;
    a.data[0] = da; a.mask[0] = ma; a.ops[0] = 0;
    a.data[1] = (op == ML_OP_MASKING || db == nullptr) ? da : db;   // B's data is never read for masking
    a.mask[1] = mb; a.ops[1] = op;
    if (op == ML_OP_UNION && esize > 0 && db == nullptr) return ml_fail(ML_ERR_ARG, "union needs B's data plane");
    return dispatch_chain(a, dc, mc, esize, n, (cudaStream_t)stream);
}

int ml_layer_chain(int64_t nlayers, const void* const* data, const uint8_t* const* mask,
                   const int32_t* ops, void* dc, uint8_t* mc, int esize, int64_t n, void* stream) {
    if (nlayers < 1 || nlayers > MAX_CHAIN) return ml_fail(ML_ERR_ARG, "chain length must be 1..16");
    ChainArgs a;
    a.nlayers = (int)nlayers;
    for (int l = 0; l < a.nlayers; ++l) {
        a.data[l] = esize > 0 ? data[l] : nullptr;
        a.mask[l] = mask[l];
        a.ops[l] = l == 0 ? (ops[0] & ML_CHAIN_EAGER) : ops[l];      // ops[0] carries flags only
        if (l > 0 && (ops[l] < ML_OP_UNION || ops[l] > ML_OP_MASKING)) return ml_fail(ML_ERR_ARG, "unknown layer operator");
    }
    return dispatch_chain(a, dc, mc, esize, n, (cudaStream_t)stream);
}

}  // extern "C"
