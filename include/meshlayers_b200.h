/*
 * meshlayers_b200.h -- C ABI of libmeshlayers_b200.so, the B200 (sm_100a) kernel backend that
 * fills the reference's compiled-backend slot `meshlayers._native`
 * (reference: pkg/setup.py:5-13 declares it; pkg/src/meshlayers/_kernels_numpy.py:3-5 makes the
 * numpy module its semantic twin).  Citations "KN:n" = _kernels_numpy.py line n, "SPEC:n" =
 * SPEC.md line n.
 *
 * Conventions
 *   - Every pointer named *_dev / plane / tri_* is a DEVICE pointer unless the function name ends
 *     in _host.  No ownership is transferred; planes are mutated in place (KN:96-99, 128-130,
 *     200-202).  Planes are row-major [row = y][col = x], y-up, texel centre = index + 0.5
 *     (KN:15, 60, 63).
 *   - `stream` is a cudaStream_t passed as void*; all work is stream-ordered, nothing synchronises
 *     the host.  Counts are written to device memory (uint64_t*), never returned by value, so a
 *     caller can batch strokes without a round trip; the *_host wrappers synchronise and return
 *     host values like the reference functions do.
 *   - Row slabs: functions taking (row0, rows) operate on rows [row0, row0+rows) of a
 *     `height`-row atlas and address planes SLAB-LOCALLY (texel (x, y) at (y-row0)*width + x).
 *     This is the multi-GPU row sharding (SPEC:150 licenses row-parallel rasterisation).
 *   - Return value: ML_OK or an ML_ERR_* code; ml_last_error() gives the message
 *     (thread-local).  The reference kernels raise nothing (KN: no validation); argument errors
 *     here correspond to TargetMismatch one layer up (errors.py:32).
 *   - tri_dtype: triangle inputs may be float32 or float64; they are widened to float64 per
 *     triangle exactly like KN:88, 113-114, 151-152.
 */
#ifndef MESHLAYERS_B200_H
#define MESHLAYERS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ML_OK = 0, ML_ERR_ARG = 1, ML_ERR_CUDA = 2, ML_ERR_NO_DEVICE = 3 };
enum { ML_F32 = 0, ML_F64 = 1 };
/* plane element kinds */
enum { ML_U8 = 0, ML_I8 = 1, ML_I16 = 2, ML_I32 = 3, ML_U32 = 4, ML_F16 = 5, ML_FLOAT32 = 6 };
/* layer algebra operators (no reference code; frozen in oracle/kn_port.c ext_layer_op) */
enum { ML_OP_UNION = 0, ML_OP_INTERSECTION = 1, ML_OP_DIFFERENCE = 2, ML_OP_MASKING = 3 };

int ml_version(void);
const char* ml_last_error(void);
/* number of SMs of the current device (148 on B200); <= 0 when no device is usable */
int ml_sm_count(void);

/* Scratch needed by every ml_raster_* / ml_coverage_fill call with `ntri` triangles. */
size_t ml_raster_workspace_bytes(int64_t ntri);

/* ---- KN:84-100  coverage_fill(tri_xy, width, height, out) -> written -------------------------
 * tri_xy [ntri][3][2] grid units.  out: uint8/bool slab.  *written (device, must be zeroed by
 * the caller) += number of texels that went 0 -> 1. */
int ml_coverage_fill(const void* tri_xy, int tri_dtype, int64_t ntri, int64_t width, int64_t height,
                     int64_t row0, int64_t rows, uint8_t* out, uint64_t* written,
                     void* workspace, size_t workspace_bytes, void* stream);

/* ---- KN:103-132  raster_depth(tri_xy, tri_zn, depth) -----------------------------------------
 * tri_xy window pixels, tri_zn [ntri][3] NDC z, depth float32 [height][width] updated in place
 * to min(depth, float32(d)) == the reference's serial result for any triangle order.  The
 * reference's returned update count depends on triangle order and is not reproduced. */
int ml_raster_depth(const void* tri_xy, const void* tri_zn, int tri_dtype, int64_t ntri,
                    float* depth, int64_t width, int64_t height,
                    void* workspace, size_t workspace_bytes, void* stream);

/* ---- KN:135-203  raster_tea(...) -> (edited, fragments) --------------------------------------
 * Scalar stroke parameters of KN:135-136.  eps_f32 != 0 reproduces numpy's float32 sum
 * depth[py,px] + eps when eps is a Python float (KN:185 under NEP-50); 0 = float64 sum. */
typedef struct ml_tea_params {
    double ww, wh;                 /* window size, KN:179-181 */
    double eps;                    /* depth bias */
    double sfx, sfy, bx, by;       /* tool map s = sfx*xn + bx, t = sfy*yn + by, KN:187-188 */
    const float* depth;            /* device, [depth_h][depth_w] */
    const uint8_t* shape;          /* device, [shape_h][shape_w], non-zero = inside tool */
    int64_t depth_w, depth_h, shape_w, shape_h;
    int32_t eps_f32;
    int32_t reserved;
} ml_tea_params;

/* Direct per-triangle TEA: exact for ANY uv layout (overlapping islands included).
 * data: slab of `esize`-byte elements (1, 2, 4); value_bits: the value already cast to the plane
 * kind, little-endian in the low bytes.  counters (device, zeroed by caller): [0] += texels whose
 * edited flag went 0 -> 1, [1] += fragments offered (KN:203). */
int ml_raster_tea(const void* tri_xy, const void* tri_clip, int tri_dtype, int64_t ntri,
                  int64_t width, int64_t height, int64_t row0, int64_t rows,
                  const ml_tea_params* params, void* data, int esize, uint32_t value_bits,
                  uint8_t* mask, uint8_t* edited, uint64_t* counters,
                  void* workspace, size_t workspace_bytes, void* stream);
/* data and mask may be NULL: the kernel then only marks the stroke's texels in `edited` (what the
 * host-buffer twin uses to bring back the written SET instead of whole planes). */

/* ---- surface map (north star (1); definition: oracle/kn_port.c ext_surface_map) ---------------
 * Pass 1: tri_id[y][x] = largest index of a triangle covering the texel centre, -1 if none.
 * counters (device, zeroed): [0] += fragments.  Overlap events (0 iff no two triangles overlap in uv
 * space) = fragments - covered texels, the latter counted by ml_surface_resolve. */
int ml_raster_tri_id(const void* tri_xy, int tri_dtype, int64_t ntri, int64_t width, int64_t height,
                     int64_t row0, int64_t rows, int32_t* tri_id, uint64_t* counters,
                     void* workspace, size_t workspace_bytes, void* stream);
/* SPEC:129-137 rasterize with a per-triangle output: out[i] = values[tri_id[i]] for every covered
 * texel whose owner triangle is kept (keep == NULL or keep[t] != 0); other texels are not touched.
 * values: [ntri] elements of esize bytes; *written (device, zeroed) += texels written. */
int ml_owner_values(const int32_t* tri_id, int64_t n, const void* values, const uint8_t* keep, int esize,
                    void* out, uint64_t* written, void* stream);
/* Pass 2: per texel, interpolate the owner triangle's attributes.  pos / nrm are three float32
 * planes each (plane stride = rows*width elements), area one float32 plane.  Uncovered texels:
 * pos = NaN, nrm = 0, area = 0.  tri_pos / tri_nrm [ntri][3][3].  *covered (device, zeroed)
 * += covered texels.  workspace: ml_surface_workspace_bytes(ntri) bytes of device scratch for the
 * per-triangle records (CCW vertices, texel area) a pre-pass writes once per call. */
int ml_surface_resolve(const void* tri_xy, const void* tri_pos, const void* tri_nrm, int tri_dtype,
                       int64_t ntri, int64_t width, int64_t row0, int64_t rows,
                       const int32_t* tri_id, float* pos, float* nrm, float* area,
                       uint64_t* covered, void* workspace, size_t workspace_bytes, void* stream);
/* Device scratch of ml_surface_resolve (64-byte per-triangle records; 16-byte aligned). */
size_t ml_surface_workspace_bytes(int64_t ntri);

/* ---- TEA over the cached triangle-id map (SURVEY.md 8 note N1) ---------------------------------
 * Bit-identical to ml_raster_tea when no two triangles overlap in uv space (overlap events == 0):
 * each covered texel re-evaluates KN:72-74 and KN:166-193 for its owner triangle.
 * tri_flags (device bitmap of (ntri+31)/32 uint32 words, may be NULL): output of ml_tea_classify
 * for THIS stroke; texels of triangles whose bit is 0 are skipped (provably unaffected).
 * worklist (device scratch, 8-byte aligned, may be NULL): when given, the id stream only COLLECTS
 * the 4-texel quads that need the float64 evaluation (24 bytes each, after a 16-byte header) and a
 * second kernel evaluates them with evenly spread parallelism; quads that do not fit are
 * evaluated in the stream kernel, so any size >= 64 bytes is valid.  Results never depend on it.
 * counters: [0] += newly edited texels, [1] += covered texels (== fragments). */
/* Footprint culling (optional, width % 128 == 0): tile_cur = the tile bitmap ml_tea_classify marked
 * for this stroke -- row segments outside it are never read, and counters[1] += known_fragments
 * (the slab's covered-texel count, which a skipping kernel cannot recount); tile_prev (may be NULL)
 * = the bitmap of the previous stroke on this `edited` plane: its tiles are cleared in the same
 * pass, which replaces the whole-plane reset of the EditedAreaMask.  Pass NULL, NULL, 0
 * to stream every texel (then the caller resets `edited` itself).
 * A tile buffer is ml_tea_tile_words() words: [bitmap | u64 count | u32 list of marked tiles].
 * tea_recs (may be NULL): per-triangle evaluation records written by ml_tea_prepare for the same
 * tri_xy / tri_clip (CCW-normalised vertices + clip coordinates as float64, 144 bytes each); with
 * them the evaluation does nine 128-bit loads per texel instead of re-deriving the winding. */
size_t ml_tea_rec_bytes(int64_t ntri);
int ml_tea_prepare(const void* tri_xy, const void* tri_clip, int tri_dtype, int64_t ntri, void* recs,
                   size_t rec_bytes, void* stream);
int ml_tea_texels(const void* tri_xy, const void* tri_clip, const void* tea_recs, int tri_dtype, int64_t ntri,
                  int64_t width, int64_t row0, int64_t rows, const int32_t* tri_id,
                  const uint32_t* tri_flags, const ml_tea_params* params, void* worklist,
                  size_t worklist_bytes, const uint32_t* tile_cur, const uint32_t* tile_prev,
                  int64_t known_fragments, void* data, int esize,
                  uint32_t value_bits, uint8_t* mask, uint8_t* edited, uint64_t* counters, void* stream);
/* Whole-atlas (no footprint culling) form of ml_tea_texels with the EditedAreaMask reset folded in:
 * reset_edited != 0 clears `edited` inside the id stream -- each quad's edited bytes are
 * zeroed by the thread that then processes the quad -- so the caller does not run a separate
 * 1 B/texel memset pass.  The id map travels through a cp.async.bulk shared-memory ring (TMA) when
 * the planes are 16-byte aligned.  known_fragments > 0 (the slab's covered-texel count, e.g. from
 * ml_surface_resolve) is reported as counters[1] instead of being recounted.  Same planes and counters as ml_tea_texels(..., NULL, NULL, 0, ...)
 * preceded by a memset of `edited`. */
int ml_tea_stream(const void* tri_xy, const void* tri_clip, const void* tea_recs, int tri_dtype, int64_t ntri,
                  int64_t width, int64_t row0, int64_t rows, const int32_t* tri_id,
                  const uint32_t* tri_flags, const ml_tea_params* params, void* worklist,
                  size_t worklist_bytes, int reset_edited, int64_t known_fragments, void* data, int esize,
                  uint32_t value_bits, uint8_t* mask, uint8_t* edited, uint64_t* counters, void* stream);
/* Per-stroke conservative triangle classification from the clip-space vertices alone:
 * bit t (bit t&31 of word t>>5) = 0 iff no fragment of triangle t can pass the w > 0, window and
 * tool-range tests (KN:174, 181, 189) -- see surface.cu for the rounding-error argument.
 * flags: (ntri+31)/32 uint32 words.  O(ntri), no texel work.
 * tile_bits (may be NULL; else ml_tea_tile_words(width, rows) words, zeroed here): additionally
 * marks every 128x8-texel tile of the slab that the raster bbox of a flagged triangle touches
 * (needs tri_xy [ntri][3][2] grid units and the slab geometry) -- the stroke's footprint. */
int ml_tea_classify(const void* tri_clip, int tri_dtype, int64_t ntri, const ml_tea_params* params,
                    uint32_t* flags, const void* tri_xy, int64_t width, int64_t height, int64_t row0,
                    int64_t rows, uint32_t* tile_bits, void* stream);
/* Same decision from the records of ml_tea_prepare: the classification then reads 16 bytes of
 * outward-rounded NDC bounds per triangle instead of the 96-byte clip record (a superset of the
 * triangles ml_tea_classify keeps, never a subset: flags stay conservative). */
int ml_tea_classify_recs(const void* tea_recs, int tri_dtype, int64_t ntri, const ml_tea_params* params,
                         uint32_t* flags, const void* tri_xy, int64_t width, int64_t height, int64_t row0,
                         int64_t rows, uint32_t* tile_bits, void* stream);
/* words of a footprint tile bitmap for a (rows x width) slab; 0 when culling is unavailable
 * (width % 128 != 0) */
int ml_tea_tile_words(int64_t width, int64_t rows);

/* ---- selection brushes (north star (2); definitions: ext_select_sphere / ext_select_threshold) -
 * Sphere brush over n texels of a position map (three float32 planes, stride pos_stride):
 * hit = ((px-cx)^2 + (py-cy)^2) + (pz-cz)^2 <= r*r in float64; hits get data = value, mask = 1,
 * edited = 1.  *count (device, zeroed) += texels whose edited flag went 0 -> 1. */
int ml_select_sphere(const float* pos, int64_t pos_stride, int64_t n,
                     double cx, double cy, double cz, double radius,
                     void* data, int esize, uint32_t value_bits, uint8_t* mask, uint8_t* edited,
                     uint64_t* count, void* stream);

/* K strokes in one pass over the position map.  Stroke k = (cx, cy, cz, r) writes value_bits[k]
 * into layer layer_of[k]; strokes are applied in index order (a later stroke overwrites an earlier
 * one on the same layer).  All arrays below are DEVICE arrays: strokes [K][4] f64, layer_of [K]
 * i32, value_bits [K] u32, data/mask/edited [L] plane pointers, counts [L] u64 (zeroed). */
int ml_select_sphere_batch(const float* pos, int64_t pos_stride, int64_t n,
                           const double* strokes, const int32_t* layer_of,
                           const uint32_t* value_bits, int64_t K,
                           void* const* data, uint8_t* const* mask, uint8_t* const* edited,
                           int64_t L, int esize, uint64_t* counts, void* stream);

/* Footprint-culled forms of the two brushes above: identical planes and counts, but a stroke reads
 * only the 128 x 4-texel tiles of the position map its sphere can reach.
 *   ml_tile_count            tiles of a (rows x width) slab; 0 when width % 128 != 0 (no culling).
 *   ml_surface_tile_boxes    once per surface map: boxes [ntiles][8] float32 (lo.xyz, 0, hi.xyz, 0;
 *                            lo > hi for a tile without covered texels), 16-byte aligned.
 *   ml_tile_workspace_bytes  device scratch (tile list) the culled brushes need, 8-byte aligned.
 * The box test is conservative (float64, margin 1e-12 relative, see select.cu box_may_hit); the
 * per-texel decision and the write rule are those of ml_select_sphere / ml_select_sphere_batch. */
int64_t ml_tile_count(int64_t width, int64_t rows);
size_t ml_tile_workspace_bytes(int64_t width, int64_t rows);
int ml_surface_tile_boxes(const float* pos, int64_t pos_stride, int64_t width, int64_t rows,
                          float* boxes, void* stream);
int ml_select_sphere_tiles(const float* pos, int64_t pos_stride, int64_t width, int64_t rows,
                           const float* boxes, void* workspace, size_t workspace_bytes,
                           double cx, double cy, double cz, double radius,
                           void* data, int esize, uint32_t value_bits, uint8_t* mask, uint8_t* edited,
                           uint64_t* count, void* stream);
int ml_select_sphere_batch_tiles(const float* pos, int64_t pos_stride, int64_t width, int64_t rows,
                                 const float* boxes, void* workspace, size_t workspace_bytes,
                                 const double* strokes, const int32_t* layer_of,
                                 const uint32_t* value_bits, int64_t K,
                                 void* const* data, uint8_t* const* mask, uint8_t* const* edited,
                                 int64_t L, int esize, uint64_t* counts, void* stream);

/* Attribute threshold: hit = (valid == NULL || valid[i] != 0) && lo <= attr[i] <= hi (closed,
 * float64 compare of the widened attribute; attr_kind is an ML_* plane kind). */
int ml_select_threshold(const void* attr, int attr_kind, const uint8_t* valid, int64_t n,
                        double lo, double hi, void* data, int esize, uint32_t value_bits,
                        uint8_t* mask, uint8_t* edited, uint64_t* count, void* stream);

/* Footprint-culled threshold selection for a float32 attribute plane that does not change between
 * selections (geometry-derived attributes such as height): ml_plane_tile_range writes [min, max] of the
 * non-NaN values per 128 x 4-texel tile (ranges [ntiles][2] float32, once per plane);
 * ml_select_threshold_tiles then reads only tiles whose range meets [lo, hi] (exact float test, no
 * margin needed) -- same planes and count as ml_select_threshold.  Scratch: ml_tile_workspace_bytes. */
int ml_plane_tile_range(const float* attr, int64_t width, int64_t rows, float* ranges, void* stream);
int ml_select_threshold_tiles(const float* attr, const uint8_t* valid, int64_t width, int64_t rows,
                              const float* ranges, void* workspace, size_t workspace_bytes,
                              double lo, double hi, void* data, int esize, uint32_t value_bits,
                              uint8_t* mask, uint8_t* edited, uint64_t* count, void* stream);

/* ---- layer algebra (north star (3); definition: ext_layer_op) ---------------------------------
 * (dc, mc) = (da, ma) op (db, mb) over n texels; mask bytes are true iff non-zero, output mask
 * bytes are exactly 0/1.  Data planes may all be NULL (esize 0, mask-only algebra: 3 B/texel).
 * Outputs may alias the A operand. */
int ml_layer_op(int op, const void* da, const uint8_t* ma, const void* db, const uint8_t* mb,
                void* dc, uint8_t* mc, int esize, int64_t n, void* stream);

/* Fused left-to-right chain  ((L0 op1 L1) op2 L2) ... op_{N-1} L_{N-1}  in one pass:
 * reads N layers, writes 1.  HOST arrays of N device pointers / N ops, N <= 16.  ops[0] is not an
 * operator: it carries flags (0, or ML_CHAIN_EAGER).  Chains of 3..8 layers read a data vector only
 * where the masks say it can contribute to the result (identical planes, fewer bytes);
 * ML_CHAIN_EAGER forces the streaming form that reads every vector of every plane. */
enum { ML_CHAIN_EAGER = 0x100 };
int ml_layer_chain(int64_t nlayers, const void* const* data, const uint8_t* const* mask,
                   const int32_t* ops, void* dc, uint8_t* mc, int esize, int64_t n, void* stream);

/* ---- per-layer area / statistics (north star (4); definitions: ext_layer_area ...) ------------
 * sums[l] (device f64, zeroed) += sum of area[i] over texels with masks[l][i] != 0, accumulated in
 * float64; counts[l] (device u64, zeroed, may be NULL) += number of such texels.  `masks` is a
 * HOST array of L device pointers (L <= 64): one pass reads area once and the L masks. */
int ml_layer_area(const float* area, const uint8_t* const* masks, int64_t L, int64_t n,
                  double* sums, uint64_t* counts, void* stream);

/* ---- fused cross-rank area reduction over peer memory (row-sharded atlases) --------
 * The reduction kernel of every rank adds its per-block partial sums / counts with SYSTEM-scope atomics into the
 * same slots of EVERY rank's result row (NVLink peer memory mapped through CUDA IPC; own row included), so the
 * all-reduce of the per-layer areas happens inside the compute kernel: no collective launch, no packing kernels.
 * Row layout (8-byte slots): [L float64 sums | L uint64 counts | uint64 arrivals | uint64 spare], zeroed before use.
 * peer_rows: HOST array of npeers device pointers (valid in THIS process) to the row of every rank for this step,
 * own row at index `self`.  arrive_table: DEVICE array of npeers pointers to the arrival slots (row + 2L) of the
 * same rows.  After the reduction kernels ONE thread signals every rank's arrival slot and waits until all npeers
 * ranks have signalled this rank's row (bounded: ~10 s without progress sets *status = 1 instead of hanging);
 * operations queued behind the call see the complete global sums in the own row.  recycle_row (may be NULL): an
 * own row to zero afterwards for a later step.  ml_peer_*: cudaMalloc'ed, zeroed regions and their 64-byte IPC
 * handles (torch's caching allocator cannot export allocation bases). */
int ml_layer_area_peers(const float* area, const uint8_t* const* masks, int64_t L, int64_t n,
                        void* const* peer_rows, int npeers, int self, void* arrive_table, uint32_t* status,
                        void* recycle_row, void* stream);
int ml_peer_alloc(void** ptr, size_t bytes);
int ml_peer_free(void* ptr);
int ml_peer_export(const void* ptr, void* handle64);
int ml_peer_open(const void* handle64, void** ptr);
int ml_peer_close(void* ptr);
/* 1 iff the current device can run native atomics on memory of device `peer_device` (NVLink peers; same device: 1) */
int ml_peer_atomics_supported(int peer_device);
/* uint8 label plane: sums[v] += area over texels with mask != 0 and data == v (v < 256). */
int ml_label_area(const float* area, const uint8_t* data, const uint8_t* mask, int64_t n,
                  double* sums /* [256] */, uint64_t* counts /* [256] */, void* stream);
/* out (device, 4 doubles): count, sum, min, max of the widened attribute over mask != 0.
 * out must be initialised to {0, 0, +inf, -inf}. */
int ml_layer_stats(const void* attr, int attr_kind, const uint8_t* mask, int64_t n,
                   double* out, void* stream);

/* ---- TPA: outline mask and padding ----------------------------------------------
 * Row-sharded stencils: the INPUT plane (cov resp. edited) is a full-width slab of global rows
 * [in_row0, in_row0+in_rows) which must contain the halo rows the rank can see; rows outside it
 * count as empty (no coverage / nothing edited).  OUTPUT planes (outline, data, mask) are slabs
 * of rows [out_row0, out_row0+out_rows), a sub-range of the input rows.
 * outline[y][x] = 1 iff cov[y][x] == 0 and some cov != 0 within Chebyshev distance <= thickness,
 * else 0. */
int ml_outline_mask(const uint8_t* cov, int64_t width, int64_t in_row0, int64_t in_rows,
                    int64_t out_row0, int64_t out_rows, int64_t thickness, uint8_t* outline,
                    void* stream);
/* padding: texels with outline != 0 within Chebyshev distance <= radius of a texel
 * with edited != 0 get data = value, mask = 1.  *count (device, zeroed) += padded texels. */
int ml_apply_padding(const uint8_t* outline, const uint8_t* edited, int64_t width,
                     int64_t in_row0, int64_t in_rows, int64_t out_row0, int64_t out_rows,
                     int64_t radius, void* data, int esize, uint32_t value_bits, uint8_t* mask,
                     uint64_t* count, void* stream);

/* Footprint-culled padding for the stroke path (single slab: input rows == output rows; width % 128
 * == 0, radius <= 4, 16-byte aligned planes): tile_bits is the 128 x 8-texel tile bitmap
 * ml_tea_classify wrote for the stroke whose `edited` marks are being padded.  Only tiles with a
 * marked tile in their 3 x 3 neighbourhood are read; planes and count equal ml_apply_padding's. */
int ml_apply_padding_tiles(const uint8_t* outline, const uint8_t* edited, int64_t width, int64_t rows,
                           int64_t radius, const uint32_t* tile_bits, void* data, int esize,
                           uint32_t value_bits, uint8_t* mask, uint64_t* count, void* stream);
/* Same, restricted to the output rows [row_lo, row_hi) of the slab.  Row-sharded atlases:
 * the `radius` rows next to a slab border need the neighbour's edited rows; the caller pads them with
 * ml_apply_padding over the exchanged halo and lets this call do the interior, so every texel is
 * visited -- and counted -- exactly once. */
int ml_apply_padding_tiles_rows(const uint8_t* outline, const uint8_t* edited, int64_t width, int64_t rows,
                                int64_t row_lo, int64_t row_hi, int64_t radius, const uint32_t* tile_bits,
                                void* data, int esize, uint32_t value_bits, uint8_t* mask, uint64_t* count,
                                void* stream);

/* ---- one call per edit: the paper's timed stroke = TEA + TPA -----------
 * ml_stroke = ml_tea_classify_recs + ml_tea_texels + ml_apply_padding_tiles on one stream, for
 * engines that keep everything resident (single slab or one rank's slab without padding halos).
 * `cur` (0 or 1) selects the tile buffer this stroke writes; the other one must be the buffer the
 * previous stroke on this `edited` plane wrote (zeroed before the first stroke) -- alternate it.
 * counters (device, 3 x u64, zeroed here): newly edited texels, fragments, padded texels. */
typedef struct ml_stroke_ctx {
    const void* tri_xy;          /* [ntri][3][2] atlas grid units */
    const void* tri_clip;        /* [ntri][3][4] clip coordinates */
    const void* tea_recs;        /* ml_tea_prepare(tri_xy, tri_clip) */
    int tri_dtype;               /* ML_F32 / ML_F64 */
    int64_t ntri;
    int64_t width, height, row0, rows;
    const int32_t* tri_id;       /* ml_raster_tri_id map of the slab */
    uint32_t* tri_flags;         /* (ntri+31)/32 words of scratch */
    void* worklist;              /* quad work list scratch (see ml_tea_texels) */
    size_t worklist_bytes;
    uint32_t* tiles[2];          /* two tile buffers of ml_tea_tile_words(width, rows) words */
    int64_t known_fragments;     /* covered texels of the slab */
    uint8_t* edited;             /* the EditedAreaMask plane */
    const uint8_t* outline;      /* outline mask for the padding pass, NULL = no TPA */
} ml_stroke_ctx;
int ml_stroke(const ml_stroke_ctx* ctx, int cur, const ml_tea_params* params, void* data, int esize,
              uint32_t value_bits, uint8_t* mask, int64_t padding_radius, uint64_t* counters, void* stream);

/* A drag gesture: n strokes (the pointer samples of SPEC:569) on one layer in ONE host call, applied in
 * order exactly like n ml_stroke calls starting with tile buffer `first_cur` (the buffers alternate;
 * after the call the next stroke uses (first_cur + n) & 1).  params / value_bits are HOST arrays of n
 * records; counters (device) receives 3 x u64 per stroke. */
int ml_stroke_sequence(const ml_stroke_ctx* ctx, int first_cur, int64_t n, const ml_tea_params* params, void* data,
                       int esize, const uint32_t* value_bits, uint8_t* mask, int64_t padding_radius,
                       uint64_t* counters, void* stream);

/* ---- display + layer file helpers (definitions: ext_resolve_display, ext_pack_mask)
 * SPEC:186-203 resolve_display: rgba_out[i] (4 bytes R,G,B,A) = mask[i] ? palette(u) : 0 with
 * u = clamp((value-lower)/(upper-lower), 0, 1), piecewise-linear over npoints control points
 * (HOST arrays: positions[npoints] strictly increasing from 0 to 1, rgba_points[npoints][4] in
 * [0,1]); channel byte = floor(c*255 + 0.5).  kind is an ML_* plane kind. */
int ml_resolve_display(const void* data, int kind, const uint8_t* mask, int64_t n,
                       double lower, double upper, const double* positions, const double* rgba_points,
                       int npoints, uint8_t* rgba_out, void* stream);
/* SPEC:221 "mask as packed bits row-major": byte plane <-> (n+7)/8 packed bytes, MSB first. */
int ml_pack_mask(const uint8_t* mask, int64_t n, uint8_t* bits, void* stream);
int ml_unpack_mask(const uint8_t* bits, int64_t n, uint8_t* mask, void* stream);

/* ---- octree baseline kernels: the remaining two callables of the reference's
 * compiled-backend slot.  float64 geometry, int32 triangle indices, uint32 cell coordinates.
 *
 * KN:303-329 expand_pairs_ordered(verts, tris, parent_cells, pair_parent, pair_tri, cube_min, child_h)
 *   -> (child_cells uint32 (M,3), child_tri int32 (M,)): every (parent cell, triangle) pair is tested
 * against the parent's 8 child cubes with the closed-box separating-axis test of KN:208-258; output
 * order is pair-major, octant-minor (octant = x | y<<1 | z<<2).  M is data dependent, so the device
 * form is two stream-ordered calls sharing `workspace`: _count writes M to *total (device), the
 * caller sizes the outputs, _emit writes them.  cube_min is a HOST array of 3 doubles. */
size_t ml_expand_pairs_workspace_bytes(int64_t npair);
int ml_expand_pairs_count(const double* verts, const int32_t* tris, const uint32_t* parent_cells,
                          const int32_t* pair_parent, const int32_t* pair_tri, int64_t npair,
                          const double* cube_min, double child_h, void* workspace, size_t workspace_bytes,
                          uint64_t* total, void* stream);
int ml_expand_pairs_emit(const uint32_t* parent_cells, const int32_t* pair_parent, const int32_t* pair_tri,
                         int64_t npair, const void* workspace, uint32_t* out_cells, int32_t* out_tri,
                         void* stream);

/* KN:361-525 raycast(origins, dirs, keys, offsets, tri_idx, verts, tris, cube_min, h, n_cells, coarse,
 *   coarse_shift, morton_encode) -> (best_t, best_tri, leaf_pos): 3D-DDA through the n_cells^3 leaf grid,
 * Moeller-Trumbore (KN:335-358) against the triangle list of every visited leaf found in the sorted
 * `keys` (nkeys Morton codes; leaf i owns tri_idx[offsets[i] .. offsets[i+1])), best hit = lexicographic
 * minimum of (t, triangle index), leaf_pos = index in `keys` of the leaf containing the hit point (-1 and
 * t = +inf on a miss).  morton_encode is fixed to the bit interleave with x in bit 0, y in bit 1, z in
 * bit 2 of every triple (n_cells <= 2^21).  coarse: optional (coarse_side^3 bytes, [x][y][z]) occupancy
 * map of the cells >> coarse_shift, NULL = none (KN:447).  cube_min is a HOST array of 3 doubles. */
int ml_raycast(const double* origins, const double* dirs, int64_t nrays, const uint64_t* keys, int64_t nkeys,
               const int64_t* offsets, const int32_t* tri_idx, const double* verts, const int32_t* tris,
               const double* cube_min, double h, int64_t n_cells, const uint8_t* coarse, int64_t coarse_side,
               int coarse_shift, double* best_t, int32_t* best_tri, int64_t* leaf_pos, void* stream);

/* Ray set-up of an octree edit ("one ray per window pixel inside the tool shape"): for the
 * nx x ny window pixels starting at (x0, y0), the ray through the pixel centre (origin on the near plane, unit
 * direction, inv_view_proj = HOST array of 16 doubles, row major) if the centre maps into a set texel of the tool
 * bitmap centred at (tool_px, tool_py) -- the tool map of KN:187-192, half open at the far edges -- and a NaN
 * direction otherwise (ml_raycast reports such a ray as a miss).  *count (device, zeroed) += rays generated. */
int ml_tool_rays(const double* inv_view_proj, int64_t cam_w, int64_t cam_h, double tool_px, double tool_py,
                 const uint8_t* shape, int64_t shape_w, int64_t shape_h, int64_t x0, int64_t y0, int64_t nx, int64_t ny,
                 double* origins, double* dirs, uint64_t* count, void* stream);

/* ---- host-buffer entry points: exact drop-ins for the reference's numpy signatures ------------
 * (KN:84 coverage_fill, KN:103 raster_depth, KN:135-136 raster_tea.)  All pointers are HOST pointers
 * to ordinary pageable memory; planes are mutated in place, counts come back through out-params, the
 * call returns when the caller's planes are final.  tri arrays are float32 or float64 (tri_dtype =
 * ML_F32 / ML_F64; the kernels widen per use like KN:88, 113, 151).
 *
 * Implementation (csrc/hostpath.cu): a persistent per-process arena (device scratch, pinned staging
 * chunks, streams, worker threads -- nothing is allocated per call once warm) and pipelined uploads.
 * coverage_fill and raster_tea never upload the caller's planes: the kernels mark the texels they
 * write in a zeroed device plane, that SET returns over PCIe as a bitmap (or as the list of its
 * non-zero 64-texel words when that is smaller) and the reference's write rule (KN:97-99, 198-202:
 * count target bytes that are 0, then store) is applied to the caller's planes by the worker threads.
 * One call at a time per process (the reference's single-writer rule); ml_host_release()
 * frees the arena. */
int ml_coverage_fill_host(const void* tri_xy, int tri_dtype, int64_t ntri, int64_t width, int64_t height,
                          uint8_t* out, int64_t* written);
int ml_raster_depth_host(const void* tri_xy, const void* tri_zn, int tri_dtype, int64_t ntri,
                         float* depth, int64_t width, int64_t height, int64_t* updated);
int ml_raster_tea_host(const void* tri_xy, const void* tri_clip, int tri_dtype, int64_t ntri,
                       double ww, double wh, const float* depth, int64_t depth_w, int64_t depth_h,
                       double eps, int eps_f32, double sfx, double sfy, double bx, double by,
                       const uint8_t* shape, int64_t shape_w, int64_t shape_h,
                       void* data, int esize, uint32_t value_bits, uint8_t* mask, uint8_t* edited,
                       int64_t width, int64_t height, int64_t* edited_count, int64_t* fragments);
void ml_host_release(void);

/* KN:303: *count = M; rows are written only when M <= capacity (re-call with a larger buffer otherwise) */
int ml_expand_pairs_ordered_host(const double* verts, int64_t nverts, const int32_t* tris, int64_t ntri,
                                 const uint32_t* parent_cells, int64_t nparents, const int32_t* pair_parent,
                                 const int32_t* pair_tri, int64_t npair, const double* cube_min, double child_h,
                                 uint32_t* out_cells, int32_t* out_tri, int64_t capacity, int64_t* count);
/* KN:361 */
int ml_raycast_host(const double* origins, const double* dirs, int64_t nrays, const uint64_t* keys, int64_t nkeys,
                    const int64_t* offsets, const int32_t* tri_idx, const double* verts, int64_t nverts,
                    const int32_t* tris, int64_t ntri, const double* cube_min, double h, int64_t n_cells,
                    const uint8_t* coarse, int64_t coarse_side, int coarse_shift,
                    double* best_t, int32_t* best_tri, int64_t* leaf_pos);

#ifdef __cplusplus
}
#endif
#endif /* MESHLAYERS_B200_H */
