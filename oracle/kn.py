"""ctypes front-end of ``oracle/kn_port.c`` -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

The three pinned functions keep the reference's positional signatures
(``_kernels_numpy.py``: ``coverage_fill`` KN:84, ``raster_depth`` KN:103, ``raster_tea``
KN:135-136): numpy arrays in, planes mutated in place, plain ints out.  Parity status of each
function is stated in the header of ``kn_port.c``.
"""
import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kn_port.c")
_LIB = os.path.join(_HERE, "_build", "libkn_port.so")

KINDS = {"uint8": 0, "int8": 1, "int16": 2, "int32": 3, "uint32": 4, "float16": 5, "float32": 6,
         "bool": 0}


def build(force=False):
    """gcc the C restatement (same -ffp-contract=off as the reference's pkg/setup.py:13)."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC",
           "-o", _LIB, _SRC, "-lm"]
    subprocess.run(cmd, check=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        i64, dbl, vp, i32 = C.c_int64, C.c_double, C.c_void_p, C.c_int
        _lib.kn_coverage_fill.restype = i64
        _lib.kn_coverage_fill.argtypes = [vp, i64, i64, i64, vp]
        _lib.kn_coverage_fill_mt.restype = i64
        _lib.kn_coverage_fill_mt.argtypes = [vp, i64, i64, i64, vp, i32]
        _lib.kn_raster_depth.restype = i64
        _lib.kn_raster_depth.argtypes = [vp, vp, i64, vp, i64, i64]
        _lib.kn_raster_depth_mt.restype = i64
        _lib.kn_raster_depth_mt.argtypes = [vp, vp, i64, vp, i64, i64, i32]
        tea = [vp, vp, i64, dbl, dbl, vp, i64, i64, dbl, i32, dbl, dbl, dbl, dbl,
               vp, i64, i64, vp, i64, vp, vp, vp, i64, i64, vp, vp]
        _lib.kn_raster_tea.restype = None
        _lib.kn_raster_tea.argtypes = tea
        _lib.kn_raster_tea_mt.restype = None
        _lib.kn_raster_tea_mt.argtypes = tea + [i32]
        _lib.kn_max_threads.restype = i32
        _lib.ext_surface_map.restype = i64
        _lib.ext_surface_map.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, vp, vp, vp, vp, vp]
        _lib.ext_surface_map_mt.restype = i64
        _lib.ext_surface_map_mt.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, vp, vp, vp, vp, vp, i32]
        _lib.ext_select_sphere_batch_fused.restype = None
        _lib.ext_select_sphere_batch_fused.argtypes = [vp, i64, i64, vp, i64, vp, vp, i64, vp, vp, vp, vp, i64, i32]
        _lib.ext_layer_chain.restype = None
        _lib.ext_layer_chain.argtypes = [i64, vp, vp, vp, vp, vp, i64, i64, i32]
        _lib.ext_layers_area.restype = None
        _lib.ext_layers_area.argtypes = [vp, vp, i64, i64, vp, vp, i32]
        _lib.ext_select_sphere.restype = i64
        _lib.ext_select_sphere.argtypes = [vp, i64, i64, dbl, dbl, dbl, dbl, vp, i64, vp, vp, vp, i32]
        _lib.ext_select_threshold.restype = i64
        _lib.ext_select_threshold.argtypes = [vp, i32, vp, i64, dbl, dbl, vp, i64, vp, vp, vp, i32]
        _lib.ext_layer_op.restype = None
        _lib.ext_layer_op.argtypes = [i32, vp, vp, vp, vp, vp, vp, i64, i64, i32]
        _lib.ext_layer_area.restype = dbl
        _lib.ext_layer_area.argtypes = [vp, vp, i64, vp, i32]
        _lib.ext_label_area.restype = None
        _lib.ext_label_area.argtypes = [vp, vp, vp, i64, vp, vp]
        _lib.ext_layer_stats.restype = None
        _lib.ext_layer_stats.argtypes = [vp, i32, vp, i64, vp, vp, vp, vp]
        _lib.ext_outline.restype = None
        _lib.ext_outline.argtypes = [vp, i64, i64, i64, vp, i32]
        _lib.ext_padding.restype = i64
        _lib.ext_padding.argtypes = [vp, vp, i64, i64, i64, vp, i64, vp, vp, i32]
        _lib.ext_mesh_surface_area.restype = dbl
        _lib.ext_mesh_surface_area.argtypes = [vp, i64]
        _lib.ext_resolve_display.restype = None
        _lib.ext_resolve_display.argtypes = [vp, i32, vp, i64, dbl, dbl, vp, vp, i32, vp]
        _lib.ext_pack_mask.restype = None
        _lib.ext_pack_mask.argtypes = [vp, i64, vp]
        _lib.kn_expand_pairs_ordered.restype = i64
        _lib.kn_expand_pairs_ordered.argtypes = [vp, vp, vp, vp, vp, i64, vp, dbl, vp, vp]
        _lib.kn_morton3.restype = C.c_uint64
        _lib.kn_morton3.argtypes = [C.c_uint64] * 3
        _lib.kn_raycast.restype = None
        _lib.kn_raycast.argtypes = [vp, vp, i64, vp, i64, vp, vp, vp, vp, vp, dbl, i64,
                                    vp, i64, i64, vp, vp, vp, i32]
    return _lib


def max_threads():
    return int(lib().kn_max_threads())


def _p(a):
    return None if a is None else a.ctypes.data


def _f64(a, shape_tail):
    """KN widens every triangle to float64 before use (KN:88, 113-114, 151-152); f32->f64 is exact."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    assert a.shape[1:] == shape_tail, (a.shape, shape_tail)
    return a


def _plane(a):
    assert isinstance(a, np.ndarray) and a.flags.c_contiguous and a.flags.writeable
    return a


def _bytes1(a):
    assert a.dtype.itemsize == 1, a.dtype
    return a


def eps_is_f32(eps):
    """numpy adds a Python float (weak scalar) to the float32 depth samples IN FLOAT32
    (KN:185, checked on numpy 2.3.5); a np.float64 scalar forces a float64 sum."""
    if isinstance(eps, np.floating):
        return eps.dtype.itemsize <= 4
    return True


def _value_bytes(value, dtype):
    return np.array(value, dtype=dtype).reshape(1).copy()


# ------------------------------------------------------------------ pinned (KN) functions

def coverage_fill(tri_xy, width, height, out, threads=0):
    tri = _f64(tri_xy, (3, 2))
    _bytes1(_plane(out))
    assert out.shape == (height, width)
    if threads:
        return int(lib().kn_coverage_fill_mt(_p(tri), tri.shape[0], width, height, _p(out), threads))
    return int(lib().kn_coverage_fill(_p(tri), tri.shape[0], width, height, _p(out)))


def raster_depth(tri_xy, tri_zn, depth, threads=0):
    tri = _f64(tri_xy, (3, 2))
    zn = _f64(tri_zn, (3,))
    assert depth.dtype == np.float32
    _plane(depth)
    h, w = depth.shape
    if threads:
        return int(lib().kn_raster_depth_mt(_p(tri), _p(zn), tri.shape[0], _p(depth), w, h, threads))
    return int(lib().kn_raster_depth(_p(tri), _p(zn), tri.shape[0], _p(depth), w, h))


def raster_tea(tri_xy, tri_clip, ww, wh, depth, eps, sfx, sfy, bx, by,
               shape, data, mask, edited, value, threads=0):
    tri = _f64(tri_xy, (3, 2))
    clip = _f64(tri_clip, (3, 4))
    depth = np.ascontiguousarray(depth)
    assert depth.dtype == np.float32
    shape = np.ascontiguousarray(shape)
    _bytes1(shape)
    _bytes1(_plane(mask))
    _bytes1(_plane(edited))
    _plane(data)
    h, w = mask.shape
    assert data.shape == (h, w) and edited.shape == (h, w)
    th, tw = shape.shape
    dh, dw = depth.shape
    assert dh >= np.ceil(wh) and dw >= np.ceil(ww), "depth plane smaller than the window"
    val = _value_bytes(value, data.dtype)
    ec = C.c_int64(0)
    fr = C.c_int64(0)
    args = [_p(tri), _p(clip), tri.shape[0], float(ww), float(wh), _p(depth), dw, dh,
            float(eps), int(eps_is_f32(eps)), float(sfx), float(sfy), float(bx), float(by),
            _p(shape), tw, th, _p(data), data.dtype.itemsize, _p(val), _p(mask), _p(edited),
            w, h, C.addressof(ec), C.addressof(fr)]
    if threads:
        lib().kn_raster_tea_mt(*args, threads)
    else:
        lib().kn_raster_tea(*args)
    return int(ec.value), int(fr.value)


def raster_tea_slab(tri_xy, tri_clip, ww, wh, depth, eps, sfx, sfy, bx, by,
                    shape, data, mask, edited, value, height, row0, threads):
    """raster_tea restricted to rows [row0, row0+rows) of a `height`-row atlas; the planes are
    slab-local (rows, width).  For CPU-baseline timing on a bounded sample of a big atlas."""
    tri = _f64(tri_xy, (3, 2))
    clip = _f64(tri_clip, (3, 4))
    depth = np.ascontiguousarray(depth, dtype=np.float32)
    shape = np.ascontiguousarray(shape)
    rows, w = mask.shape
    th, tw = shape.shape
    dh, dw = depth.shape
    val = _value_bytes(value, data.dtype)
    ec, fr = C.c_int64(0), C.c_int64(0)
    f = lib().kn_raster_tea_slab
    f.restype = None
    f.argtypes = lib().kn_raster_tea.argtypes[:-2] + [C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_int]
    f(_p(tri), _p(clip), tri.shape[0], float(ww), float(wh), _p(depth), dw, dh, float(eps),
      int(eps_is_f32(eps)), float(sfx), float(sfy), float(bx), float(by), _p(shape), tw, th,
      _p(_plane(data)), data.dtype.itemsize, _p(val), _p(_plane(mask)), _p(_plane(edited)), w, height,
      row0, row0 + rows, C.addressof(ec), C.addressof(fr), threads)
    return int(ec.value), int(fr.value)


# ------------------------------------------------------------------ extension definitions

def surface_map(tri_xy, tri_pos, tri_nrm, width, height, rows=None, threads=0):
    """Returns dict(tri_id, pos[3,h,w], nrm[3,h,w], area, covered, overlap) for rows [r0,r1).
    threads > 0: row-parallel form (same arrays)."""
    tri = _f64(tri_xy, (3, 2))
    P = _f64(tri_pos, (3, 3))
    N = _f64(tri_nrm, (3, 3))
    r0, r1 = rows if rows is not None else (0, height)
    n = r1 - r0
    tri_id = np.empty((n, width), np.int32)
    pos = np.empty((3, n, width), np.float32)
    nrm = np.empty((3, n, width), np.float32)
    area = np.empty((n, width), np.float32)
    ov = C.c_int64(0)
    if threads:
        cov = lib().ext_surface_map_mt(_p(tri), _p(P), _p(N), tri.shape[0], width, height, r0, r1,
                                       _p(tri_id), _p(pos), _p(nrm), _p(area), C.addressof(ov), threads)
    else:
        cov = lib().ext_surface_map(_p(tri), _p(P), _p(N), tri.shape[0], width, height, r0, r1,
                                    _p(tri_id), _p(pos), _p(nrm), _p(area), C.addressof(ov))
    return dict(tri_id=tri_id, pos=pos, nrm=nrm, area=area, covered=int(cov), overlap=int(ov.value))


def select_sphere(pos, center, radius, data, mask, edited, value, threads=1):
    assert pos.dtype == np.float32 and pos.flags.c_contiguous and pos.shape[0] == 3
    n = mask.size
    assert pos[0].size == n
    val = _value_bytes(value, data.dtype)
    return int(lib().ext_select_sphere(_p(pos), n, n, float(center[0]), float(center[1]),
                                       float(center[2]), float(radius), _p(_plane(data)),
                                       data.dtype.itemsize, _p(val), _p(_bytes1(_plane(mask))),
                                       _p(_bytes1(_plane(edited))), threads))


def _ptr_array(arrs):
    return (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def select_sphere_batch(pos, strokes, layer_of, values, data, mask, edited, threads=1):
    """K strokes (rows of `strokes` = cx, cy, cz, r) in ONE pass; stroke k writes values[k] into layer
    layer_of[k] of the plane lists.  Returns the per-layer edited counts (int64 array, len(data))."""
    assert pos.dtype == np.float32 and pos.flags.c_contiguous and pos.shape[0] == 3
    L = len(data)
    n = mask[0].size
    assert pos[0].size == n
    strokes = np.ascontiguousarray(strokes, np.float64).reshape(-1, 4)
    K = strokes.shape[0]
    lo = np.ascontiguousarray(layer_of, np.int32)
    vals = np.ascontiguousarray(np.asarray(values).astype(data[0].dtype)).reshape(K)
    for a in list(data) + list(mask) + list(edited):
        _plane(a)
    counts = np.zeros(L, np.int64)
    lib().ext_select_sphere_batch_fused(_p(pos), n, n, _p(strokes), K, _p(lo), _ptr_array(data),
                                        data[0].dtype.itemsize, _p(vals.view(np.uint8)), _ptr_array(mask),
                                        _ptr_array(edited), _p(counts), L, threads)
    return counts


def select_threshold(attr, valid, lo, hi, data, mask, edited, value, threads=1):
    attr = np.ascontiguousarray(attr)
    kind = KINDS[attr.dtype.name]
    n = mask.size
    assert attr.size == n
    if valid is not None:
        valid = np.ascontiguousarray(valid)
        _bytes1(valid)
    val = _value_bytes(value, data.dtype)
    return int(lib().ext_select_threshold(_p(attr), kind, _p(valid), n, float(lo), float(hi),
                                          _p(_plane(data)), data.dtype.itemsize, _p(val),
                                          _p(_bytes1(_plane(mask))), _p(_bytes1(_plane(edited))),
                                          threads))


OPS = {"union": 0, "intersection": 1, "difference": 2, "masking": 3}


def layer_op(op, da, ma, db, mb, dc, mc, threads=1):
    """(dc, mc) = (da, ma) <op> (db, mb); data planes may all be None (mask-only algebra)."""
    n = ma.size
    es = 0 if da is None else da.dtype.itemsize
    lib().ext_layer_op(OPS[op], _p(da), _p(_bytes1(ma)), _p(db), _p(_bytes1(mb)), _p(dc),
                       _p(_bytes1(_plane(mc))), es, n, threads)


def layer_chain(ops, data, mask, dc, mc, threads=1):
    """Fused left fold ((L0 op0 L1) op1 L2) ... in one pass; `data` may be None (mask-only)."""
    nl = len(mask)
    assert len(ops) == nl - 1
    code = np.array([OPS[o] for o in ops], np.int32)
    es = 0 if data is None else data[0].dtype.itemsize
    for m in mask:
        assert m.flags.c_contiguous
        _bytes1(m)
    lib().ext_layer_chain(nl, _p(code), None if data is None else _ptr_array(data), _ptr_array(mask),
                          _p(dc), _p(_bytes1(_plane(mc))), es, mask[0].size, threads)


def layers_area(area, masks, threads=1):
    """Areas and texel counts of several layers in one pass: (float64[L], int64[L])."""
    assert area.dtype == np.float32
    area = np.ascontiguousarray(area)
    L = len(masks)
    sums, counts = np.zeros(L, np.float64), np.zeros(L, np.int64)
    keep = [_bytes1(np.ascontiguousarray(m)) for m in masks]          # keeps any copy alive across the call
    lib().ext_layers_area(_p(area), _ptr_array(keep), L, masks[0].size, _p(sums), _p(counts), threads)
    return sums, counts


def layer_area(area, mask, threads=1):
    assert area.dtype == np.float32
    cnt = C.c_int64(0)
    a = lib().ext_layer_area(_p(np.ascontiguousarray(area)), _p(_bytes1(np.ascontiguousarray(mask))),
                             mask.size, C.addressof(cnt), threads)
    return float(a), int(cnt.value)


def label_area(area, data, mask):
    assert area.dtype == np.float32 and data.dtype.itemsize == 1
    out = np.zeros(256, np.float64)
    cnt = np.zeros(256, np.int64)
    lib().ext_label_area(_p(np.ascontiguousarray(area)), _p(np.ascontiguousarray(data)),
                         _p(np.ascontiguousarray(mask)), mask.size, _p(out), _p(cnt))
    return out, cnt


def layer_stats(attr, mask):
    attr = np.ascontiguousarray(attr)
    cnt = C.c_int64(0)
    s, mn, mx = C.c_double(0), C.c_double(0), C.c_double(0)
    lib().ext_layer_stats(_p(attr), KINDS[attr.dtype.name], _p(np.ascontiguousarray(mask)), mask.size,
                          C.addressof(cnt), C.addressof(s), C.addressof(mn), C.addressof(mx))
    return int(cnt.value), float(s.value), float(mn.value), float(mx.value)


def outline(cov, thickness, threads=1):
    cov = np.ascontiguousarray(cov)
    out = np.zeros(cov.shape, np.uint8)
    h, w = cov.shape
    lib().ext_outline(_p(_bytes1(cov)), w, h, int(thickness), _p(out), threads)
    return out


def padding(outline_mask, edited, radius, data, mask, value, threads=1):
    h, w = mask.shape
    val = _value_bytes(value, data.dtype)
    return int(lib().ext_padding(_p(_bytes1(np.ascontiguousarray(outline_mask))),
                                 _p(_bytes1(np.ascontiguousarray(edited))), w, h, int(radius),
                                 _p(_plane(data)), data.dtype.itemsize, _p(val),
                                 _p(_bytes1(_plane(mask))), threads))


def mesh_surface_area(tri_pos):
    P = _f64(tri_pos, (3, 3))
    return float(lib().ext_mesh_surface_area(_p(P), P.shape[0]))


def resolve_display(data, mask, lower, upper, positions, colours):
    """(h, w, 4) uint8 RGBA plane of a layer (definition of SPEC.md:195-203 used by the GPU tests)."""
    data = np.ascontiguousarray(data)
    mask = np.ascontiguousarray(mask)
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    col = np.ascontiguousarray(colours, dtype=np.float64).reshape(-1, 4)
    out = np.zeros(mask.shape + (4,), np.uint8)
    lib().ext_resolve_display(_p(data), KINDS[data.dtype.name], _p(_bytes1(mask)), mask.size, float(lower), float(upper),
                              _p(pos), _p(col), len(pos), _p(out))
    return out


def pack_mask(mask):
    mask = np.ascontiguousarray(mask)
    out = np.zeros((mask.size + 7) // 8, np.uint8)
    lib().ext_pack_mask(_p(_bytes1(mask)), mask.size, _p(out))
    return out


def morton_encode(x, y, z):
    """The key convention of the octree kernels: bit interleave, x in bit 0, y in bit 1, z in
    bit 2 of every triple (the octant code of KN:267).  numpy, vectorised; this is the callable
    a caller hands to the reference's ``raycast`` (KN:362)."""
    def spread(v):
        v = np.asarray(v).astype(np.uint64) & np.uint64(0x1fffff)
        v = (v | (v << np.uint64(32))) & np.uint64(0x1f00000000ffff)
        v = (v | (v << np.uint64(16))) & np.uint64(0x1f0000ff0000ff)
        v = (v | (v << np.uint64(8))) & np.uint64(0x100f00f00f00f00f)
        v = (v | (v << np.uint64(4))) & np.uint64(0x10c30c30c30c30c3)
        v = (v | (v << np.uint64(2))) & np.uint64(0x1249249249249249)
        return v
    return spread(x) | (spread(y) << np.uint64(1)) | (spread(z) << np.uint64(2))


def expand_pairs_ordered(verts, tris, parent_cells, pair_parent, pair_tri, cube_min, child_h):
    """KN:303-329, same positional signature and return value."""
    npair = int(np.asarray(pair_parent).shape[0])
    verts = np.ascontiguousarray(verts, np.float64)
    tris = np.ascontiguousarray(tris, np.int64)
    pc = np.ascontiguousarray(parent_cells, np.int64).reshape(-1, 3)
    pp = np.ascontiguousarray(pair_parent, np.int64)
    pt = np.ascontiguousarray(pair_tri, np.int64)
    cm = np.ascontiguousarray(cube_min, np.float64)
    cells = np.zeros((8 * npair, 3), np.uint32)
    tri = np.zeros(8 * npair, np.int32)
    m = lib().kn_expand_pairs_ordered(_p(verts), _p(tris), _p(pc), _p(pp), _p(pt), npair, _p(cm),
                                      float(child_h), _p(cells), _p(tri))
    return cells[:m].copy(), tri[:m].copy()


def raycast(origins, dirs, keys, offsets, tri_idx, verts, tris, cube_min, h, n_cells, coarse,
            coarse_shift, morton_encode=None, threads=1):
    """KN:361-525, same positional signature and return value (float64 inputs; the Morton
    convention is fixed, see ``morton_encode`` above)."""
    origins = np.ascontiguousarray(origins, np.float64)
    dirs = np.ascontiguousarray(dirs, np.float64)
    keys = np.ascontiguousarray(keys, np.uint64)
    offsets = np.ascontiguousarray(offsets, np.int64)
    tri_idx = np.ascontiguousarray(tri_idx, np.int32)
    verts = np.ascontiguousarray(verts, np.float64)
    tris = np.ascontiguousarray(tris, np.int64)
    cm = np.ascontiguousarray(cube_min, np.float64)
    n = origins.shape[0]
    cz = None if coarse is None else np.ascontiguousarray(coarse != 0, np.uint8)
    best_t = np.empty(n, np.float64)
    best_tri = np.empty(n, np.int32)
    leaf = np.empty(n, np.int64)
    lib().kn_raycast(_p(origins), _p(dirs), n, _p(keys), keys.shape[0], _p(offsets), _p(tri_idx),
                     _p(verts), _p(tris), _p(cm), float(h), int(n_cells), _p(cz),
                     0 if cz is None else cz.shape[0], int(coarse_shift or 0),
                     _p(best_t), _p(best_tri), _p(leaf), int(threads))
    return best_t, best_tri, leaf
