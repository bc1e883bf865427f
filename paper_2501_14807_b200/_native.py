"""``_native`` -- the compiled kernel backend, B200 edition.

This module fills the slot the reference declares as ``meshlayers._native`` (reference
``pkg/setup.py:5-13``): the function-for-function twin of ``meshlayers._kernels_numpy`` (KN).
The three hot functions keep KN's names, positional signatures, in-place plane mutation and
return conventions:

    coverage_fill(tri_xy, width, height, out) -> int                       KN:84
    raster_depth(tri_xy, tri_zn, depth) -> int                             KN:103
    raster_tea(tri_xy, tri_clip, ww, wh, depth, eps, sfx, sfy, bx, by,
               shape, data, mask, edited, value) -> (int, int)             KN:135-136

and so do the two octree-baseline kernels (the paper's competitor):

    expand_pairs_ordered(verts, tris, parent_cells, pair_parent, pair_tri,
                         cube_min, child_h) -> (cells, tri)                KN:303
    raycast(origins, dirs, keys, offsets, tri_idx, verts, tris, cube_min, h,
            n_cells, coarse, coarse_shift, morton_encode) -> (t, tri, leaf) KN:361

They accept either numpy arrays (HOST buffers, exactly like the reference: the call uploads,
runs the CUDA kernels, downloads the planes in place) or torch CUDA tensors (device resident:
nothing is copied).  Everything below them is an extension for the north-star operations
(surface map, sphere / threshold selection, layer algebra, areas, outline / padding) and works
on torch CUDA tensors only.

All compute happens in ``libmeshlayers_b200.so`` (hand-written sm_100a CUDA behind the C ABI of
``include/meshlayers_b200.h``), loaded with ctypes.  There is NO CPU fallback: if the library
or a CUDA device is missing every call raises ``BackendUnavailable``.
"""
import ctypes as C
import math
import os

import numpy as np

from .errors import BackendUnavailable, MeshLayersError, TargetMismatch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmeshlayers_b200.so")

ML_F32, ML_F64 = 0, 1
KIND_CODES = {"uint8": 0, "bool": 0, "int8": 1, "int16": 2, "int32": 3, "uint32": 4,
              "float16": 5, "float32": 6}
OPS = {"union": 0, "intersection": 1, "difference": 2, "masking": 3}

_lib = None


class _TeaParams(C.Structure):
    _fields_ = [("ww", C.c_double), ("wh", C.c_double), ("eps", C.c_double),
                ("sfx", C.c_double), ("sfy", C.c_double), ("bx", C.c_double), ("by", C.c_double),
                ("depth", C.c_void_p), ("shape", C.c_void_p),
                ("depth_w", C.c_int64), ("depth_h", C.c_int64),
                ("shape_w", C.c_int64), ("shape_h", C.c_int64),
                ("eps_f32", C.c_int32), ("reserved", C.c_int32)]


class _StrokeCtx(C.Structure):
    """include/meshlayers_b200.h ml_stroke_ctx."""
    _fields_ = [("tri_xy", C.c_void_p), ("tri_clip", C.c_void_p), ("tea_recs", C.c_void_p),
                ("tri_dtype", C.c_int), ("ntri", C.c_int64),
                ("width", C.c_int64), ("height", C.c_int64), ("row0", C.c_int64), ("rows", C.c_int64),
                ("tri_id", C.c_void_p), ("tri_flags", C.c_void_p), ("worklist", C.c_void_p),
                ("worklist_bytes", C.c_size_t), ("tiles", C.c_void_p * 2), ("known_fragments", C.c_int64),
                ("edited", C.c_void_p), ("outline", C.c_void_p)]


def lib():
    """Load the C-ABI library (once).  Raises BackendUnavailable when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise BackendUnavailable(
            "libmeshlayers_b200.so is not built; run `python -m paper_2501_14807_b200.build` "
            "(there is no CPU fallback)")
    try:
        L = C.CDLL(LIB_PATH)
    except OSError as exc:                                   # pragma: no cover
        raise BackendUnavailable("cannot load %s: %s" % (LIB_PATH, exc))
    i64, i32, dbl, vp, u32, sz = C.c_int64, C.c_int, C.c_double, C.c_void_p, C.c_uint32, C.c_size_t
    sig = {
        "ml_version": (i32, []),
        "ml_last_error": (C.c_char_p, []),
        "ml_sm_count": (i32, []),
        "ml_raster_workspace_bytes": (sz, [i64]),
        "ml_coverage_fill": (i32, [vp, i32, i64, i64, i64, i64, i64, vp, vp, vp, sz, vp]),
        "ml_raster_depth": (i32, [vp, vp, i32, i64, vp, i64, i64, vp, sz, vp]),
        "ml_raster_tea": (i32, [vp, vp, i32, i64, i64, i64, i64, i64, C.POINTER(_TeaParams), vp, i32,
                                u32, vp, vp, vp, vp, sz, vp]),
        "ml_raster_tri_id": (i32, [vp, i32, i64, i64, i64, i64, i64, vp, vp, vp, sz, vp]),
        "ml_surface_resolve": (i32, [vp, vp, vp, i32, i64, i64, i64, i64, vp, vp, vp, vp, vp, vp, sz, vp]),
        "ml_surface_workspace_bytes": (sz, [i64]),
        "ml_owner_values": (i32, [vp, i64, vp, vp, i32, vp, vp, vp]),
        "ml_tea_texels": (i32, [vp, vp, vp, i32, i64, i64, i64, i64, vp, vp, C.POINTER(_TeaParams), vp, sz,
                                vp, vp, i64, vp, i32, u32, vp, vp, vp, vp]),
        "ml_tea_stream": (i32, [vp, vp, vp, i32, i64, i64, i64, i64, vp, vp, C.POINTER(_TeaParams), vp, sz,
                                i32, i64, vp, i32, u32, vp, vp, vp, vp]),
        "ml_tea_classify_recs": (i32, [vp, i32, i64, C.POINTER(_TeaParams), vp, vp, i64, i64, i64, i64, vp, vp]),
        "ml_stroke": (i32, [C.POINTER(_StrokeCtx), i32, C.POINTER(_TeaParams), vp, i32, u32, vp, i64, vp, vp]),
        "ml_stroke_sequence": (i32, [C.POINTER(_StrokeCtx), i32, i64, C.POINTER(_TeaParams), vp, i32, C.POINTER(C.c_uint32), vp,
                                     i64, vp, vp]),
        "ml_tea_rec_bytes": (sz, [i64]),
        "ml_tea_prepare": (i32, [vp, vp, i32, i64, vp, sz, vp]),
        "ml_tea_classify": (i32, [vp, i32, i64, C.POINTER(_TeaParams), vp, vp, i64, i64, i64, i64, vp, vp]),
        "ml_tea_tile_words": (i32, [i64, i64]),
        "ml_select_sphere": (i32, [vp, i64, i64, dbl, dbl, dbl, dbl, vp, i32, u32, vp, vp, vp, vp]),
        "ml_select_sphere_batch": (i32, [vp, i64, i64, vp, vp, vp, i64, vp, vp, vp, i64, i32, vp, vp]),
        "ml_tile_count": (i64, [i64, i64]),
        "ml_tile_workspace_bytes": (sz, [i64, i64]),
        "ml_surface_tile_boxes": (i32, [vp, i64, i64, i64, vp, vp]),
        "ml_select_sphere_tiles": (i32, [vp, i64, i64, i64, vp, vp, sz, dbl, dbl, dbl, dbl, vp, i32, u32, vp, vp,
                                         vp, vp]),
        "ml_select_sphere_batch_tiles": (i32, [vp, i64, i64, i64, vp, vp, sz, vp, vp, vp, i64, vp, vp, vp, i64,
                                               i32, vp, vp]),
        "ml_select_threshold": (i32, [vp, i32, vp, i64, dbl, dbl, vp, i32, u32, vp, vp, vp, vp]),
        "ml_plane_tile_range": (i32, [vp, i64, i64, vp, vp]),
        "ml_select_threshold_tiles": (i32, [vp, vp, i64, i64, vp, vp, sz, dbl, dbl, vp, i32, u32, vp, vp, vp, vp]),
        "ml_layer_op": (i32, [i32, vp, vp, vp, vp, vp, vp, i32, i64, vp]),
        "ml_layer_chain": (i32, [i64, vp, vp, vp, vp, vp, i32, i64, vp]),
        "ml_layer_area": (i32, [vp, vp, i64, i64, vp, vp, vp]),
        "ml_layer_area_peers": (i32, [vp, vp, i64, i64, vp, i32, i32, vp, vp, vp, vp]),
        "ml_peer_alloc": (i32, [C.POINTER(vp), sz]),
        "ml_peer_free": (i32, [vp]),
        "ml_peer_export": (i32, [vp, vp]),
        "ml_peer_open": (i32, [vp, C.POINTER(vp)]),
        "ml_peer_close": (i32, [vp]),
        "ml_peer_atomics_supported": (i32, [i32]),
        "ml_label_area": (i32, [vp, vp, vp, i64, vp, vp, vp]),
        "ml_layer_stats": (i32, [vp, i32, vp, i64, vp, vp]),
        "ml_outline_mask": (i32, [vp, i64, i64, i64, i64, i64, i64, vp, vp]),
        "ml_apply_padding": (i32, [vp, vp, i64, i64, i64, i64, i64, i64, vp, i32, u32, vp, vp, vp]),
        "ml_apply_padding_tiles": (i32, [vp, vp, i64, i64, i64, vp, vp, i32, u32, vp, vp, vp]),
        "ml_apply_padding_tiles_rows": (i32, [vp, vp, i64, i64, i64, i64, i64, vp, vp, i32, u32, vp, vp, vp]),
        "ml_resolve_display": (i32, [vp, i32, vp, i64, dbl, dbl, vp, vp, i32, vp, vp]),
        "ml_pack_mask": (i32, [vp, i64, vp, vp]),
        "ml_unpack_mask": (i32, [vp, i64, vp, vp]),
        "ml_coverage_fill_host": (i32, [vp, i32, i64, i64, i64, vp, vp]),
        "ml_raster_depth_host": (i32, [vp, vp, i32, i64, vp, i64, i64, vp]),
        "ml_raster_tea_host": (i32, [vp, vp, i32, i64, dbl, dbl, vp, i64, i64, dbl, i32, dbl, dbl, dbl, dbl,
                                     vp, i64, i64, vp, i32, u32, vp, vp, i64, i64, vp, vp]),
        "ml_host_release": (None, []),
        "ml_expand_pairs_workspace_bytes": (sz, [i64]),
        "ml_expand_pairs_count": (i32, [vp, vp, vp, vp, vp, i64, vp, dbl, vp, sz, vp, vp]),
        "ml_expand_pairs_emit": (i32, [vp, vp, vp, i64, vp, vp, vp, vp]),
        "ml_raycast": (i32, [vp, vp, i64, vp, i64, vp, vp, vp, vp, vp, dbl, i64, vp, i64, i32, vp, vp, vp, vp]),
        "ml_tool_rays": (i32, [vp, i64, i64, dbl, dbl, vp, i64, i64, i64, i64, i64, i64, vp, vp, vp, vp]),
        "ml_expand_pairs_ordered_host": (i32, [vp, i64, vp, i64, vp, i64, vp, vp, i64, vp, dbl, vp, vp, i64, vp]),
        "ml_raycast_host": (i32, [vp, vp, i64, vp, i64, vp, vp, vp, i64, vp, i64, vp, dbl, i64, vp, i64, i32,
                                  vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


EXPORTED_SYMBOLS = (
    "ml_version", "ml_last_error", "ml_sm_count", "ml_raster_workspace_bytes", "ml_coverage_fill",
    "ml_raster_depth", "ml_raster_tea", "ml_raster_tri_id", "ml_surface_resolve",
    "ml_surface_workspace_bytes", "ml_owner_values", "ml_tea_texels", "ml_tea_stream", "ml_tea_rec_bytes", "ml_tea_prepare",
    "ml_tea_classify_recs", "ml_stroke", "ml_stroke_sequence",
    "ml_tea_classify", "ml_tea_tile_words", "ml_select_sphere", "ml_select_sphere_batch", "ml_tile_count",
    "ml_tile_workspace_bytes", "ml_surface_tile_boxes", "ml_select_sphere_tiles", "ml_select_sphere_batch_tiles",
    "ml_select_threshold", "ml_plane_tile_range", "ml_select_threshold_tiles", "ml_layer_op",
    "ml_layer_chain", "ml_layer_area", "ml_layer_area_peers", "ml_peer_alloc", "ml_peer_free", "ml_peer_export",
    "ml_peer_open", "ml_peer_close", "ml_peer_atomics_supported", "ml_label_area", "ml_layer_stats", "ml_outline_mask",
    "ml_apply_padding", "ml_apply_padding_tiles", "ml_apply_padding_tiles_rows", "ml_resolve_display", "ml_pack_mask", "ml_unpack_mask",
    "ml_coverage_fill_host", "ml_raster_depth_host", "ml_raster_tea_host", "ml_host_release",
    "ml_expand_pairs_workspace_bytes", "ml_expand_pairs_count", "ml_expand_pairs_emit", "ml_raycast",
    "ml_expand_pairs_ordered_host", "ml_raycast_host", "ml_tool_rays")


def _check(rc):
    if rc == 0:
        return
    msg = lib().ml_last_error().decode("utf-8", "replace")
    if rc == 1:
        raise TargetMismatch(msg)
    if rc == 3:
        raise BackendUnavailable(msg)
    raise MeshLayersError("libmeshlayers_b200: " + msg)


def _torch():
    import torch
    return torch


_cuda_checked = False


def require_cuda():
    """Fail loudly when the CUDA path cannot run (no fallback exists).  The positive answer is
    cached: this sits on the per-stroke path."""
    global _cuda_checked
    torch = _torch()
    if not _cuda_checked:
        if not torch.cuda.is_available():
            raise BackendUnavailable("no CUDA device visible; paper_2501_14807_b200 has no CPU fallback")
        lib()
        _cuda_checked = True
    return torch


def _is_cuda_tensor(a):
    return type(a).__module__.startswith("torch") and hasattr(a, "is_cuda") and a.is_cuda


def _stream():
    """Raw handle of torch's current stream on the current device.  ``torch.cuda.current_stream()``
    costs ~15 us per call (three per stroke); the raw accessor it wraps costs well under 1 us."""
    torch = _torch()
    try:
        return C.c_void_p(torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()))
    except AttributeError:                                    # pragma: no cover - older / newer torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _tri_dev(a, tail, device):
    """Triangle attribute array -> contiguous CUDA tensor of float32/float64 (widened on device
    per triangle like KN:88).  numpy inputs are uploaded."""
    torch = _torch()
    if not _is_cuda_tensor(a):
        a = np.ascontiguousarray(a)
        if a.dtype not in (np.float32, np.float64):
            a = a.astype(np.float64)
        a = torch.from_numpy(a).to(device)
    if a.dtype not in (torch.float32, torch.float64):
        a = a.to(torch.float64)
    a = a.contiguous()
    if tuple(a.shape[1:]) != tail:
        raise TargetMismatch("expected triangle array of shape (T,%s), got %s" % (tail, tuple(a.shape)))
    return a, (ML_F32 if a.dtype == torch.float32 else ML_F64)


def _same_dtype(*arrs):
    torch = _torch()
    if len({a.dtype for a in arrs}) > 1:
        return [a.to(torch.float64) for a in arrs]
    return list(arrs)


def _np_dtype_of(t):
    """numpy dtype with the same element layout as a torch tensor / numpy array."""
    if isinstance(t, np.ndarray):
        return t.dtype
    name = str(t.dtype).replace("torch.", "")
    return np.dtype("bool" if name == "bool" else name)


def value_bits(value, plane):
    """Cast ``value`` the way numpy casts a scalar stored into the plane (KN:200) and return the
    element's bytes as an unsigned integer."""
    dt = _np_dtype_of(plane)
    if dt.itemsize not in (1, 2, 4):
        raise TargetMismatch("data plane element size %d not supported" % dt.itemsize)
    v = np.array(value, dtype=dt).reshape(1)
    return int(v.view({1: np.uint8, 2: np.uint16, 4: np.uint32}[dt.itemsize])[0]), dt.itemsize


def _byte_plane(t, what):
    if _np_dtype_of(t).itemsize != 1:
        raise TargetMismatch("%s plane must have 1-byte elements (bool / uint8)" % what)
    if not t.is_contiguous():
        raise TargetMismatch("%s plane must be contiguous" % what)
    return t


def eps_is_f32(eps):
    """KN:185 adds ``eps`` to float32 depth samples: numpy keeps the sum in float32 for a Python
    float (weak scalar) or np.float32, and promotes to float64 for np.float64."""
    if isinstance(eps, np.floating):
        return eps.dtype.itemsize <= 4
    return True


def _workspace(ntri, device):
    torch = _torch()
    nbytes = int(lib().ml_raster_workspace_bytes(int(ntri)))
    return torch.empty(nbytes, dtype=torch.uint8, device=device), nbytes


def _counters(n, device):
    torch = _torch()
    return torch.zeros(n, dtype=torch.int64, device=device)


# =============================================================================================
# KN twins
# =============================================================================================

def _tri_host(*arrays):
    """Host triangle arrays as the host twins take them: C-contiguous, all float32 (when every input
    is float32 -- half the PCIe bytes) or all float64.  Returns (arrays..., ML dtype code)."""
    f32 = all(isinstance(a, np.ndarray) and a.dtype == np.float32 for a in arrays)
    dt = np.float32 if f32 else np.float64
    return tuple(np.ascontiguousarray(a, dtype=dt) for a in arrays) + (ML_F32 if f32 else ML_F64,)


def coverage_fill(tri_xy, width, height, out, *, row0=0, counts=None):
    """KN:84-100.  ``out``: (rows, width) uint8/bool plane, numpy (host) or torch CUDA (device).
    Returns the number of texels that went 0 -> 1 (or None when ``counts`` is supplied)."""
    L = lib()
    if isinstance(out, np.ndarray):
        if out.shape != (height, width) or out.dtype.itemsize != 1 or not out.flags.c_contiguous:
            raise TargetMismatch("out must be a contiguous (height, width) uint8 plane")
        tri, dt = _tri_host(tri_xy)
        if tri.shape[1:] != (3, 2):
            raise TargetMismatch("tri_xy must be (T,3,2)")
        written = C.c_int64(0)
        _check(L.ml_coverage_fill_host(tri.ctypes.data, dt, tri.shape[0], width, height,
                                       out.ctypes.data, C.addressof(written)))
        return int(written.value)
    require_cuda()
    _byte_plane(out, "out")
    rows = out.shape[0]
    if out.shape[1] != width or row0 < 0 or row0 + rows > height:
        raise TargetMismatch("out slab does not fit a %dx%d plane" % (height, width))
    tri, dt = _tri_dev(tri_xy, (3, 2), out.device)
    ws, nb = _workspace(tri.shape[0], out.device)
    ctr = counts if counts is not None else _counters(2, out.device)
    _check(L.ml_coverage_fill(_ptr(tri), dt, tri.shape[0], width, height, row0, rows, _ptr(out),
                              _ptr(ctr), _ptr(ws), nb, _stream()))
    return None if counts is not None else int(ctr[0].item())


def raster_depth(tri_xy, tri_zn, depth, *, count=True):
    """KN:103-132.  ``depth``: (Wh, Ww) float32 plane updated in place.  The reference's return
    value depends on triangle order; this returns the number of texels whose
    depth changed instead.  ``count=False`` (device planes) skips that count -- it costs a copy of
    the plane and a host read-back -- and returns None."""
    L = lib()
    if isinstance(depth, np.ndarray):
        if depth.dtype != np.float32 or depth.ndim != 2 or not depth.flags.c_contiguous:
            raise TargetMismatch("depth must be a contiguous 2-D float32 plane")
        tri, zn, dt = _tri_host(tri_xy, tri_zn)
        if tri.shape[1:] != (3, 2) or zn.shape != (tri.shape[0], 3):
            raise TargetMismatch("tri_xy must be (T,3,2) and tri_zn (T,3)")
        upd = C.c_int64(0)
        h, w = depth.shape
        _check(L.ml_raster_depth_host(tri.ctypes.data, zn.ctypes.data, dt, tri.shape[0],
                                      depth.ctypes.data, w, h, C.addressof(upd)))
        return int(upd.value)
    torch = require_cuda()
    if depth.dtype != torch.float32 or depth.dim() != 2 or not depth.is_contiguous():
        raise TargetMismatch("depth must be a contiguous 2-D float32 plane")
    tri, _ = _tri_dev(tri_xy, (3, 2), depth.device)
    zn, _ = _tri_dev(tri_zn, (3,), depth.device)
    tri, zn = _same_dtype(tri, zn)
    dt = ML_F32 if tri.dtype == torch.float32 else ML_F64
    if zn.shape[0] != tri.shape[0]:
        raise TargetMismatch("tri_xy / tri_zn triangle counts differ")
    before = depth.clone() if count else None
    ws, nb = _workspace(tri.shape[0], depth.device)
    h, w = depth.shape
    _check(L.ml_raster_depth(_ptr(tri), _ptr(zn), dt, tri.shape[0], _ptr(depth), w, h,
                             _ptr(ws), nb, _stream()))
    if not count:
        return None
    return int((before.view(torch.int32) != depth.view(torch.int32)).sum().item())


def _tea_params(ww, wh, depth, eps, sfx, sfy, bx, by, shape):
    p = _TeaParams()
    p.ww, p.wh, p.eps = float(ww), float(wh), float(eps)
    p.sfx, p.sfy, p.bx, p.by = float(sfx), float(sfy), float(bx), float(by)
    p.depth, p.shape = depth.data_ptr(), shape.data_ptr()
    p.depth_h, p.depth_w = depth.shape
    p.shape_h, p.shape_w = shape.shape
    p.eps_f32 = int(eps_is_f32(eps))
    return p


def _check_window(ww, wh, depth_shape, shape_shape):
    if not (depth_shape[0] >= math.ceil(wh) and depth_shape[1] >= math.ceil(ww)):
        raise TargetMismatch("depth plane %s smaller than the %sx%s window" % (tuple(depth_shape), ww, wh))
    if shape_shape[0] < 1 or shape_shape[1] < 1:
        raise TargetMismatch("tool shape plane is empty")


def raster_tea(tri_xy, tri_clip, ww, wh, depth, eps, sfx, sfy, bx, by,
               shape, data, mask, edited, value, *, height=None, row0=0, counts=None):
    """KN:135-203, direct per-triangle kernel.  Returns (edited_texels, fragments_offered)."""
    L = lib()
    if isinstance(mask, np.ndarray):
        h, w = mask.shape
        if data.shape != (h, w) or edited.shape != (h, w):
            raise TargetMismatch("data / mask / edited planes disagree in shape")
        for a, nm in ((data, "data"), (mask, "mask"), (edited, "edited")):
            if not a.flags.c_contiguous:
                raise TargetMismatch(nm + " plane must be C-contiguous")
        if mask.dtype.itemsize != 1 or edited.dtype.itemsize != 1:
            raise TargetMismatch("mask / edited planes must be bool or uint8")
        tri, clip, dt = _tri_host(tri_xy, tri_clip)
        if tri.shape[1:] != (3, 2) or clip.shape != (tri.shape[0], 3, 4):
            raise TargetMismatch("tri_xy must be (T,3,2) and tri_clip (T,3,4)")
        dep = np.ascontiguousarray(depth, dtype=np.float32)
        shp = np.ascontiguousarray(shape)
        if shp.dtype.itemsize != 1:
            shp = (shp != 0).astype(np.uint8)
        _check_window(ww, wh, dep.shape, shp.shape)
        bits, esize = value_bits(value, data)
        ec, fr = C.c_int64(0), C.c_int64(0)
        _check(L.ml_raster_tea_host(tri.ctypes.data, clip.ctypes.data, dt, tri.shape[0], float(ww), float(wh),
                                    dep.ctypes.data, dep.shape[1], dep.shape[0], float(eps),
                                    int(eps_is_f32(eps)), float(sfx), float(sfy), float(bx), float(by),
                                    shp.ctypes.data, shp.shape[1], shp.shape[0], data.ctypes.data, esize,
                                    bits, mask.ctypes.data, edited.ctypes.data, w, h,
                                    C.addressof(ec), C.addressof(fr)))
        return int(ec.value), int(fr.value)
    torch = require_cuda()
    rows, w = mask.shape
    height = rows if height is None else height
    if tuple(data.shape) != (rows, w) or tuple(edited.shape) != (rows, w):
        raise TargetMismatch("data / mask / edited planes disagree in shape")
    _byte_plane(mask, "mask")
    _byte_plane(edited, "edited")
    if not data.is_contiguous():
        raise TargetMismatch("data plane must be contiguous")
    dev = mask.device
    tri, _ = _tri_dev(tri_xy, (3, 2), dev)
    clip, _ = _tri_dev(tri_clip, (3, 4), dev)
    tri, clip = _same_dtype(tri, clip)
    dt = ML_F32 if tri.dtype == torch.float32 else ML_F64
    depth = _as_dev(depth, torch.float32, dev)
    shape = _as_dev_bytes(shape, dev)
    _check_window(ww, wh, depth.shape, shape.shape)
    p = _tea_params(ww, wh, depth, eps, sfx, sfy, bx, by, shape)
    bits, esize = value_bits(value, data)
    ws, nb = _workspace(tri.shape[0], dev)
    ctr = counts if counts is not None else _counters(2, dev)
    _check(L.ml_raster_tea(_ptr(tri), _ptr(clip), dt, tri.shape[0], w, height, row0, rows, C.byref(p),
                           _ptr(data), esize, bits, _ptr(mask), _ptr(edited), _ptr(ctr), _ptr(ws), nb,
                           _stream()))
    if counts is not None:
        return None
    c = ctr.tolist()
    return int(c[0]), int(c[1])


def _as_dev(a, dtype, device):
    torch = _torch()
    if not _is_cuda_tensor(a):
        a = torch.from_numpy(np.ascontiguousarray(a)).to(device)
    if a.dtype != dtype:
        a = a.to(dtype)
    return a.contiguous()


def _as_dev_bytes(a, device):
    torch = _torch()
    if not _is_cuda_tensor(a):
        a = np.ascontiguousarray(a)
        if a.dtype.itemsize != 1:
            a = (a != 0).astype(np.uint8)
        a = torch.from_numpy(a.view(np.uint8)).to(device)
    elif _np_dtype_of(a).itemsize != 1:
        a = (a != 0).to(torch.uint8)
    return a.contiguous()


# ---- octree baseline kernels (KN:303, KN:361) -------------------------------------------------

def morton_encode(x, y, z):
    """The Morton convention compiled into ``raycast``: bit interleave with x in bit 0, y in bit 1,
    z in bit 2 of every triple (the octant code of KN:267), 21 bits per axis.  This is the callable
    to hand to the reference's ``raycast`` (KN:362) when comparing; numpy arrays or torch tensors."""
    if _is_cuda_tensor(x) or type(x).__module__.startswith("torch"):
        torch = _torch()

        def spread(v):
            v = v.to(torch.int64) & 0x1fffff
            for sh, m in ((32, 0x1f00000000ffff), (16, 0x1f0000ff0000ff), (8, 0x100f00f00f00f00f),
                          (4, 0x10c30c30c30c30c3), (2, 0x1249249249249249)):
                v = (v | (v << sh)) & m
            return v
        return spread(x) | (spread(y) << 1) | (spread(z) << 2)         # int64: 63 bits are enough

    def spread(v):
        v = np.asarray(v).astype(np.uint64) & np.uint64(0x1fffff)
        for sh, m in ((32, 0x1f00000000ffff), (16, 0x1f0000ff0000ff), (8, 0x100f00f00f00f00f),
                      (4, 0x10c30c30c30c30c3), (2, 0x1249249249249249)):
            v = (v | (v << np.uint64(sh))) & np.uint64(m)
        return v
    return spread(x) | (spread(y) << np.uint64(1)) | (spread(z) << np.uint64(2))


_MORTON_PROBE = (np.array([1, 0, 0, 5, 65535, 2], np.uint64), np.array([0, 1, 0, 3, 1, 40000], np.uint64),
                 np.array([0, 0, 1, 6, 7, 9], np.uint64))


def _check_morton(fn):
    """``raycast`` takes the key function as an argument in the reference (KN:362); the kernel has one
    convention compiled in, so a different callable must fail loudly instead of missing every leaf."""
    if fn is None or fn is morton_encode:
        return
    got = np.asarray(fn(*_MORTON_PROBE)).astype(np.uint64)
    if not np.array_equal(got, morton_encode(*_MORTON_PROBE)):
        raise TargetMismatch("raycast: morton_encode differs from the compiled convention "
                             "(bit interleave, x lowest; see _native.morton_encode)")


def _host_array(a, dtype, tail=None):
    a = np.ascontiguousarray(a, dtype=dtype)
    if tail is not None and a.shape[1:] != tail:
        raise TargetMismatch("expected an array of shape (N,%s), got %s" % (tail, a.shape))
    return a


def _dev_array(a, dtype, device, tail=None):
    torch = _torch()
    if not _is_cuda_tensor(a):
        a = np.ascontiguousarray(a)
        if a.dtype.kind == "u" and a.dtype.itemsize > 1:              # torch has no arithmetic on them
            a = a.astype(np.int64)
        a = torch.from_numpy(a).to(device)
    a = a.to(dtype).contiguous()
    if tail is not None and tuple(a.shape[1:]) != tail:
        raise TargetMismatch("expected an array of shape (N,%s), got %s" % (tail, tuple(a.shape)))
    return a


def _cube_min3(cube_min):
    cm = cube_min.detach().cpu().numpy() if hasattr(cube_min, "detach") else cube_min
    cm = np.ascontiguousarray(cm, dtype=np.float64).reshape(-1)
    if cm.shape[0] != 3:
        raise TargetMismatch("cube_min must have 3 components")
    return cm


def expand_pairs_ordered(verts, tris, parent_cells, pair_parent, pair_tri, cube_min, child_h, *,
                         max_rows=None):
    """KN:303-329: refine (parent cell, triangle) pairs one octree level down; returns
    ``(child_cells uint32 (M,3), child_tri int32 (M,))`` pair-major, octant-minor.  numpy inputs
    (HOST buffers, like the reference) return numpy arrays; if ``pair_tri`` is a torch CUDA tensor
    everything stays on the device and torch tensors come back (cells as int32: coordinates are
    below 2^21, so the bits equal the reference's uint32).
    Geometry is widened to float64 exactly as KN:312-324 does before its first arithmetic.
    ``max_rows`` (device form): raise ``MemoryBudgetExceeded`` before allocating more output rows."""
    L = lib()
    cm = _cube_min3(cube_min)
    if not _is_cuda_tensor(pair_tri):
        v = _host_array(verts, np.float64, (3,))
        t = _host_array(tris, np.int32, (3,))
        pc = _host_array(parent_cells, np.uint32, (3,))
        pp = _host_array(pair_parent, np.int32)
        pt = _host_array(pair_tri, np.int32)
        npair = pp.shape[0]
        if pt.shape[0] != npair:
            raise TargetMismatch("pair_parent / pair_tri lengths differ")
        cap = min(8 * npair, max(2 * npair, 4096))
        count = C.c_int64(0)
        while True:
            cells = np.empty((cap, 3), np.uint32)
            tri = np.empty(cap, np.int32)
            _check(L.ml_expand_pairs_ordered_host(v.ctypes.data, v.shape[0], t.ctypes.data, t.shape[0],
                                                  pc.ctypes.data, pc.shape[0], pp.ctypes.data, pt.ctypes.data,
                                                  npair, cm.ctypes.data, float(child_h), cells.ctypes.data,
                                                  tri.ctypes.data, cap, C.addressof(count)))
            if count.value <= cap:
                break
            cap = int(count.value)
        return cells[:count.value].copy(), tri[:count.value].copy()
    torch = require_cuda()
    dev = pair_tri.device
    v = _dev_array(verts, torch.float64, dev, (3,))
    t = _dev_array(tris, torch.int32, dev, (3,))
    pc = _dev_array(parent_cells, torch.int32, dev, (3,))
    pp = _dev_array(pair_parent, torch.int32, dev)
    pt = _dev_array(pair_tri, torch.int32, dev)
    npair = pp.shape[0]
    if pt.shape[0] != npair:
        raise TargetMismatch("pair_parent / pair_tri lengths differ")
    nb = int(L.ml_expand_pairs_workspace_bytes(npair))
    ws = torch.empty(nb, dtype=torch.uint8, device=dev)
    total = torch.zeros(1, dtype=torch.int64, device=dev)
    _check(L.ml_expand_pairs_count(_ptr(v), _ptr(t), _ptr(pc), _ptr(pp), _ptr(pt), npair, cm.ctypes.data,
                                   float(child_h), _ptr(ws), nb, _ptr(total), _stream()))
    m = int(total.item())
    if max_rows is not None and m > max_rows:
        from .errors import MemoryBudgetExceeded
        raise MemoryBudgetExceeded("octree level needs %d (cell, triangle) rows, the budget allows %d"
                                   % (m, max_rows))
    cells = torch.empty((m, 3), dtype=torch.int32, device=dev)        # coordinates < 2^21: int32 == uint32
    tri = torch.empty(m, dtype=torch.int32, device=dev)
    if m:
        _check(L.ml_expand_pairs_emit(_ptr(pc), _ptr(pp), _ptr(pt), npair, _ptr(ws), _ptr(cells), _ptr(tri),
                                      _stream()))
    return cells, tri


def raycast(origins, dirs, keys, offsets, tri_idx, verts, tris, cube_min, h, n_cells, coarse,
            coarse_shift, morton_encode=None):
    """KN:361-525: march every ray front to back through the leaf grid; returns
    ``(best_t float64, best_tri int32, leaf_pos int64)``.  numpy inputs return numpy arrays, torch CUDA
    ``origins`` keep everything on the device.  float64 geometry (the reference would compute partly in
    float32 for float32 inputs, KN:340, 381; such inputs are widened first here).  ``morton_encode`` must
    be the compiled convention (``_native.morton_encode``) or None."""
    L = lib()
    _check_morton(morton_encode)
    cm = _cube_min3(cube_min)
    n_cells = int(n_cells)
    shift = int(coarse_shift or 0)
    if coarse is not None and (coarse.ndim != 3 or len(set(coarse.shape)) != 1):
        raise TargetMismatch("coarse must be a cubic 3-D occupancy array")
    if not _is_cuda_tensor(origins):
        o = _host_array(origins, np.float64, (3,))
        d = _host_array(dirs, np.float64, (3,))
        k = _host_array(keys, np.uint64)
        off = _host_array(offsets, np.int64)
        idx = _host_array(tri_idx, np.int32)
        v = _host_array(verts, np.float64, (3,))
        t = _host_array(tris, np.int32, (3,))
        if d.shape != o.shape or off.shape[0] != k.shape[0] + 1:
            raise TargetMismatch("raycast: origins/dirs or keys/offsets shapes disagree")
        cz = None if coarse is None else np.ascontiguousarray(np.asarray(coarse) != 0, dtype=np.uint8)
        n = o.shape[0]
        best_t = np.full(n, np.inf)
        best_tri = np.full(n, -1, np.int32)
        leaf = np.full(n, -1, np.int64)
        _check(L.ml_raycast_host(o.ctypes.data, d.ctypes.data, n, k.ctypes.data, k.shape[0], off.ctypes.data,
                                 idx.ctypes.data, v.ctypes.data, v.shape[0], t.ctypes.data, t.shape[0],
                                 cm.ctypes.data, float(h), n_cells, None if cz is None else cz.ctypes.data,
                                 0 if cz is None else cz.shape[0], shift, best_t.ctypes.data,
                                 best_tri.ctypes.data, leaf.ctypes.data))
        return best_t, best_tri, leaf
    torch = require_cuda()
    dev = origins.device
    o = _dev_array(origins, torch.float64, dev, (3,))
    d = _dev_array(dirs, torch.float64, dev, (3,))
    if _is_cuda_tensor(keys) and keys.dtype in (torch.int64, torch.uint64):
        k = keys.contiguous()
    else:
        k = torch.from_numpy(np.ascontiguousarray(keys, dtype=np.uint64).view(np.int64)).to(dev)
    off = _dev_array(offsets, torch.int64, dev)
    idx = _dev_array(tri_idx, torch.int32, dev)
    v = _dev_array(verts, torch.float64, dev, (3,))
    t = _dev_array(tris, torch.int32, dev, (3,))
    if d.shape != o.shape or off.shape[0] != k.shape[0] + 1:
        raise TargetMismatch("raycast: origins/dirs or keys/offsets shapes disagree")
    cz = None
    if coarse is not None:
        cz = coarse if _is_cuda_tensor(coarse) else torch.from_numpy(np.ascontiguousarray(coarse)).to(dev)
        cz = (cz != 0).to(torch.uint8).contiguous()
    n = o.shape[0]
    best_t = torch.empty(n, dtype=torch.float64, device=dev)
    best_tri = torch.empty(n, dtype=torch.int32, device=dev)
    leaf = torch.empty(n, dtype=torch.int64, device=dev)
    _check(L.ml_raycast(_ptr(o), _ptr(d), n, _ptr(k), k.shape[0], _ptr(off), _ptr(idx), _ptr(v), _ptr(t),
                        cm.ctypes.data, float(h), n_cells, _ptr(cz), 0 if cz is None else cz.shape[0], shift,
                        _ptr(best_t), _ptr(best_tri), _ptr(leaf), _stream()))
    return best_t, best_tri, leaf


# =============================================================================================
# Extensions (torch CUDA tensors only)
# =============================================================================================

def surface_map(tri_xy, tri_pos, tri_nrm, width, height, *, row0=0, rows=None, device=None):
    """Texture-space rasterisation of the mesh into the per-texel surface map (north star (1);
    definition oracle/kn_port.c ext_surface_map).  Returns a dict of CUDA tensors:
    tri_id int32 (rows,width); pos, nrm float32 (3,rows,width); area float32 (rows,width); and
    ints covered, fragments, overlap (= fragments - covered; 0 iff no uv overlap)."""
    torch = require_cuda()
    L = lib()
    device = torch.device(device or "cuda")
    rows = height - row0 if rows is None else rows
    tri, _ = _tri_dev(tri_xy, (3, 2), device)
    P, _ = _tri_dev(tri_pos, (3, 3), device)
    N, _ = _tri_dev(tri_nrm, (3, 3), device)
    tri, P, N = _same_dtype(tri, P, N)
    dt = ML_F32 if tri.dtype == torch.float32 else ML_F64
    T = tri.shape[0]
    if P.shape[0] != T or N.shape[0] != T:
        raise TargetMismatch("triangle attribute arrays disagree in length")
    tri_id = torch.empty((rows, width), dtype=torch.int32, device=device)
    pos = torch.empty((3, rows, width), dtype=torch.float32, device=device)
    nrm = torch.empty((3, rows, width), dtype=torch.float32, device=device)
    area = torch.empty((rows, width), dtype=torch.float32, device=device)
    ctr = _counters(3, device)
    ws, nb = _workspace(T, device)
    _check(L.ml_raster_tri_id(_ptr(tri), dt, T, width, height, row0, rows, _ptr(tri_id), _ptr(ctr),
                              _ptr(ws), nb, _stream()))
    sb = int(L.ml_surface_workspace_bytes(T))
    recs = torch.empty(sb, dtype=torch.uint8, device=device)       # per-triangle records, freed after the build
    _check(L.ml_surface_resolve(_ptr(tri), _ptr(P), _ptr(N), dt, T, width, row0, rows, _ptr(tri_id),
                                _ptr(pos), _ptr(nrm), _ptr(area), C.c_void_p(ctr.data_ptr() + 16),
                                _ptr(recs), sb, _stream()))
    c = ctr.tolist()
    return dict(tri_id=tri_id, pos=pos, nrm=nrm, area=area, fragments=int(c[0]), overlap=int(c[0]) - int(c[2]),
                covered=int(c[2]))


def raster_tri_id(tri_xy, width, height, *, row0=0, rows=None, device=None):
    """Pass 1 of the surface map only.  Returns (tri_id, fragments, overlap)."""
    torch = require_cuda()
    device = torch.device(device or "cuda")
    rows = height - row0 if rows is None else rows
    tri, dt = _tri_dev(tri_xy, (3, 2), device)
    tri_id = torch.empty((rows, width), dtype=torch.int32, device=device)
    ctr = _counters(2, device)
    ws, nb = _workspace(tri.shape[0], device)
    _check(lib().ml_raster_tri_id(_ptr(tri), dt, tri.shape[0], width, height, row0, rows, _ptr(tri_id),
                                  _ptr(ctr), _ptr(ws), nb, _stream()))
    fragments = int(ctr[0].item())
    return tri_id, fragments, fragments - int((tri_id >= 0).sum().item())       # overlap = fragments - covered


def owner_values(tri_id, values, out, keep=None):
    """out[texel] = values[owner triangle] for covered texels (optionally only kept triangles).
    Returns the number of texels written."""
    torch = require_cuda()
    if tuple(tri_id.shape) != tuple(out.shape) or not out.is_contiguous():
        raise TargetMismatch("target plane does not match the triangle-id map")
    esize = _np_dtype_of(out).itemsize
    if _np_dtype_of(values).itemsize != esize or not values.is_contiguous():
        raise TargetMismatch("per-triangle values must have the target's element kind")
    ctr = _counters(1, tri_id.device)
    _check(lib().ml_owner_values(_ptr(tri_id), tri_id.numel(), _ptr(values), _ptr(keep), esize, _ptr(out), _ptr(ctr),
                                 _stream()))
    return int(ctr[0].item())


def tea_texels(tri_xy, tri_clip, tri_id, ww, wh, depth, eps, sfx, sfy, bx, by,
               shape, data, mask, edited, value, *, row0=0, counts=None, classify=True, scratch=None,
               height=None, tiles=None, known_fragments=0, recs=None, reset_edited=False):
    """TEA over the cached triangle-id map (SURVEY.md 8 note N1): same planes and counts as
    ``raster_tea`` when the uv layout has no overlaps.  Returns (edited_texels, fragments).
    ``classify`` runs the per-stroke triangle pre-pass (ml_tea_classify) so that texels of
    triangles outside the tool footprint skip the float64 evaluation; results are identical
    either way.  ``tiles=(cur, prev)`` (int32 tensors of ``tea_tile_words`` words, ``prev`` may be
    None) switches on footprint culling: only tiles a flagged triangle's raster bbox touches are
    read, the tiles of ``prev`` (the previous stroke's ``cur``) have their ``edited`` bytes
    cleared, and ``known_fragments`` (the slab's covered texel count) is reported as fragments.
    The caller must then NOT reset ``edited`` itself and must pass ``height``.  ``recs`` (from
    ``tea_prepare`` for the same triangle arrays) makes the evaluation read one prepared 144-byte
    record per triangle instead of re-deriving the winding per texel (identical result).
    ``reset_edited`` (whole-atlas form only, i.e. without ``tiles``): the kernel clears ``edited``
     while it streams the id map, instead of the caller running a memset pass first."""
    torch = require_cuda()
    rows, w = mask.shape
    dev = mask.device
    if tuple(tri_id.shape) != (rows, w) or tuple(data.shape) != (rows, w) or tuple(edited.shape) != (rows, w):
        raise TargetMismatch("tri_id / data / mask / edited planes disagree in shape")
    _byte_plane(mask, "mask")
    _byte_plane(edited, "edited")
    tri, _ = _tri_dev(tri_xy, (3, 2), dev)
    clip, _ = _tri_dev(tri_clip, (3, 4), dev)
    tri, clip = _same_dtype(tri, clip)
    dt = ML_F32 if tri.dtype == torch.float32 else ML_F64
    depth = _as_dev(depth, torch.float32, dev)
    shape = _as_dev_bytes(shape, dev)
    _check_window(ww, wh, depth.shape, shape.shape)
    p = _tea_params(ww, wh, depth, eps, sfx, sfy, bx, by, shape)
    bits, esize = value_bits(value, data)
    ctr = counts if counts is not None else _counters(2, dev)
    flags = work = None
    if classify:
        # scratch = (triangle bitmap int32[(T+31)/32], worklist int64[...]) may be supplied to avoid
        # per-stroke allocation
        if scratch is None:
            scratch = tea_scratch(tri.shape[0], rows * w, dev)
        flags, work = scratch
        cur = tiles[0] if tiles else None
        if cur is not None and not classify:
            raise TargetMismatch("footprint culling needs the classification pass")
        hh = int(height if height is not None else row0 + rows)
        if recs is not None:          # 16-byte prepared bounds per triangle instead of the 96-byte clip record
            _check(lib().ml_tea_classify_recs(_ptr(recs), dt, tri.shape[0], C.byref(p), _ptr(flags), _ptr(tri), w,
                                              hh, row0, rows, _ptr(cur), _stream()))
        else:
            _check(lib().ml_tea_classify(_ptr(clip), dt, tri.shape[0], C.byref(p), _ptr(flags), _ptr(tri), w,
                                         hh, row0, rows, _ptr(cur), _stream()))
    cur, prev = tiles if tiles else (None, None)
    if reset_edited and cur is not None:
        raise TargetMismatch("reset_edited belongs to the whole-atlas form; culled strokes clear their footprint tiles")
    if cur is None and (reset_edited or os.environ.get("ML_TEA_STREAM_ENTRY")):
        _check(lib().ml_tea_stream(_ptr(tri), _ptr(clip), _ptr(recs), dt, tri.shape[0], w, row0, rows, _ptr(tri_id),
                                   _ptr(flags), C.byref(p), _ptr(work), 0 if work is None else work.numel() * 8,
                                   1 if reset_edited else 0, int(known_fragments), _ptr(data), esize, bits, _ptr(mask), _ptr(edited),
                                   _ptr(ctr), _stream()))
        if counts is not None:
            return None
        c = ctr.tolist()
        return int(c[0]), int(c[1])
    _check(lib().ml_tea_texels(_ptr(tri), _ptr(clip), _ptr(recs), dt, tri.shape[0], w, row0, rows, _ptr(tri_id),
                               _ptr(flags), C.byref(p), _ptr(work), 0 if work is None else work.numel() * 8,
                               _ptr(cur), _ptr(prev), int(known_fragments),
                               _ptr(data), esize, bits, _ptr(mask), _ptr(edited), _ptr(ctr), _stream()))
    if counts is not None:
        return None
    c = ctr.tolist()
    return int(c[0]), int(c[1])


def tea_prepare(tri_xy, tri_clip, device=None):
    """Per-triangle records of the TEA evaluation (CCW-normalised uv vertices + clip coordinates in
    float64), valid while the triangle arrays and the camera do not change."""
    torch = require_cuda()
    dev = torch.device(device or tri_xy.device)
    tri, _ = _tri_dev(tri_xy, (3, 2), dev)
    clip, _ = _tri_dev(tri_clip, (3, 4), dev)
    tri, clip = _same_dtype(tri, clip)
    dt = ML_F32 if tri.dtype == torch.float32 else ML_F64
    nb = int(lib().ml_tea_rec_bytes(tri.shape[0]))
    recs = torch.empty(nb, dtype=torch.uint8, device=dev)
    _check(lib().ml_tea_prepare(_ptr(tri), _ptr(clip), dt, tri.shape[0], _ptr(recs), nb, _stream()))
    return recs


def stroke_ctx(tri_xy, tri_clip, recs, tri_id, flags, worklist, tiles, edited, outline, *, width, height, row0,
               rows, known_fragments):
    """Fill an ``ml_stroke_ctx`` for ``stroke_call`` (all arguments are resident CUDA tensors; the
    caller keeps them alive)."""
    torch = _torch()
    c = _StrokeCtx()
    c.tri_xy, c.tri_clip, c.tea_recs = tri_xy.data_ptr(), tri_clip.data_ptr(), recs.data_ptr()
    c.tri_dtype = ML_F32 if tri_xy.dtype == torch.float32 else ML_F64
    c.ntri = tri_xy.shape[0]
    c.width, c.height, c.row0, c.rows = int(width), int(height), int(row0), int(rows)
    c.tri_id, c.tri_flags = tri_id.data_ptr(), flags.data_ptr()
    c.worklist, c.worklist_bytes = worklist.data_ptr(), worklist.numel() * 8
    c.tiles[0], c.tiles[1] = tiles[0].data_ptr(), tiles[1].data_ptr()
    c.known_fragments = int(known_fragments)
    c.edited = edited.data_ptr()
    c.outline = outline.data_ptr() if outline is not None else None
    return c


def stroke_call(cstruct, cur, ww, wh, depth, eps, sfx, sfy, bx, by, shape, data, mask, value, radius, counts):
    """One C call per edit (``ml_stroke``): classification, TEA and padding on the current stream.
    ``counts`` (int64[3], device) receives edited / fragments / padded."""
    shape = _as_dev_bytes(shape, data.device)
    _check_window(ww, wh, depth.shape, shape.shape)
    p = _tea_params(ww, wh, depth, eps, sfx, sfy, bx, by, shape)
    bits, esize = value_bits(value, data)
    _check(lib().ml_stroke(C.byref(cstruct), int(cur), C.byref(p), _ptr(data), esize, bits, _ptr(mask), int(radius),
                           _ptr(counts), _stream()))


def stroke_sequence_call(cstruct, first_cur, ww, wh, depth, eps, tool_maps, shapes, data, mask, values, radius, counts):
    """``ml_stroke_sequence``: n strokes in one C call.  ``tool_maps`` = n tuples (sfx, sfy, bx, by),
    ``shapes`` = n device shape planes, ``values`` = n stroke values, ``counts`` int64[n,3] on the device."""
    n = len(tool_maps)
    params = (_TeaParams * n)()
    vbits = (C.c_uint32 * n)()
    esize = 1
    alive = []                     # uploaded shape planes must outlive the queued kernels of ALL strokes
    for k in range(n):
        shape = _as_dev_bytes(shapes[k], data.device)
        alive.append(shape)
        _check_window(ww, wh, depth.shape, shape.shape)
        params[k] = _tea_params(ww, wh, depth, eps, *tool_maps[k], shape)
        vbits[k], esize = value_bits(values[k], data)
    _check(lib().ml_stroke_sequence(C.byref(cstruct), int(first_cur), n, params, _ptr(data), esize, vbits, _ptr(mask),
                                    int(radius), _ptr(counts), _stream()))


def tea_scratch(ntri, ntexels, device, max_quads=1 << 24):
    """Per-stroke scratch of ``tea_texels``: triangle flags and the quad work list (device)."""
    torch = _torch()
    cap = max(8, min((ntexels + 3) // 4, max_quads))
    return (torch.empty(max(1, (ntri + 31) // 32), dtype=torch.int32, device=device),
            torch.empty(2 + 3 * cap, dtype=torch.int64, device=device))


def tea_tile_words(width, rows):
    """Words of a footprint tile bitmap for a slab; 0 when culling is unavailable (width % 128)."""
    return int(lib().ml_tea_tile_words(int(width), int(rows)))


def _check_layer_planes(n, data, mask, edited):
    if mask.numel() != n or data.numel() != n or (edited is not None and edited.numel() != n):
        raise TargetMismatch("layer planes do not match the %d-texel map" % n)
    _byte_plane(mask, "mask")
    if edited is not None:
        _byte_plane(edited, "edited")
    if not data.is_contiguous():
        raise TargetMismatch("data plane must be contiguous")


class TileBoxes:
    """Bounding boxes of the position map per 128 x 4-texel tile plus the tile-list scratch the
    footprint-culled brushes use (one per surface map; ``None`` from ``tile_boxes`` when the slab
    width is not a multiple of 128)."""

    def __init__(self, boxes, scratch, nbytes):
        self.boxes, self.scratch, self.nbytes = boxes, scratch, nbytes


def tile_boxes(pos):
    """Build the per-tile position boxes of a (3, rows, width) float32 position map."""
    torch = require_cuda()
    L = lib()
    rows, width = int(pos.shape[1]), int(pos.shape[2])
    nt = int(L.ml_tile_count(width, rows))
    if nt == 0 or pos.data_ptr() % 16 or (rows * width) % 4:
        return None
    boxes = torch.empty((nt, 8), dtype=torch.float32, device=pos.device)
    _check(L.ml_surface_tile_boxes(_ptr(pos), rows * width, width, rows, _ptr(boxes), _stream()))
    nb = int(L.ml_tile_workspace_bytes(width, rows))
    return TileBoxes(boxes, torch.empty(nb, dtype=torch.uint8, device=pos.device), nb)


def select_sphere(pos, center, radius, data, mask, edited, value, *, counts=None, tiles=None):
    """Sphere brush over a (3, rows, width) float32 position map.  Returns newly edited texels.
    ``tiles`` (a TileBoxes of this position map) selects the footprint-culled kernels: same
    planes and count, but only the tiles the sphere can reach are read."""
    torch = require_cuda()
    if pos.dtype != torch.float32 or pos.dim() != 3 or pos.shape[0] != 3 or not pos.is_contiguous():
        raise TargetMismatch("pos must be a contiguous (3, rows, width) float32 tensor")
    n = pos.shape[1] * pos.shape[2]
    _check_layer_planes(n, data, mask, edited)
    bits, esize = value_bits(value, data)
    ctr = counts if counts is not None else _counters(1, pos.device)
    aligned = all(t.data_ptr() % 16 == 0 for t in (data, mask, edited))
    if tiles is not None and aligned:
        _check(lib().ml_select_sphere_tiles(_ptr(pos), n, int(pos.shape[2]), int(pos.shape[1]), _ptr(tiles.boxes),
                                            _ptr(tiles.scratch), tiles.nbytes, float(center[0]), float(center[1]),
                                            float(center[2]), float(radius), _ptr(data), esize, bits, _ptr(mask),
                                            _ptr(edited), _ptr(ctr), _stream()))
    else:
        _check(lib().ml_select_sphere(_ptr(pos), n, n, float(center[0]), float(center[1]), float(center[2]),
                                      float(radius), _ptr(data), esize, bits, _ptr(mask), _ptr(edited),
                                      _ptr(ctr), _stream()))
    return None if counts is not None else int(ctr[0].item())


class StrokeBatch:
    """Device-resident description of K sphere strokes over L layers (pointer tables included),
    reusable across calls: the only per-step host->device traffic is the stroke record upload."""

    RECORD_BYTES = 40                    # per stroke: 4 x float64 (cx, cy, cz, r) + int32 layer + uint32 value bits

    def __init__(self, layers_data, layers_mask, layers_edited, device, capacity=0):
        torch = _torch()
        self.L = len(layers_data)
        self.data, self.mask, self.edited = list(layers_data), list(layers_mask), list(layers_edited)
        esizes = {_np_dtype_of(d).itemsize for d in self.data}
        if len(esizes) != 1:
            raise TargetMismatch("all layers of a batch must share one element size")
        self.esize = esizes.pop()
        if any(t.data_ptr() % 16 or not t.is_contiguous() for t in self.data + self.mask + self.edited):
            raise TargetMismatch("batched strokes need contiguous, 16-byte aligned layer planes")
        mk = lambda ts: torch.tensor([t.data_ptr() for t in ts], dtype=torch.int64, device=device)
        self.d_data, self.d_mask, self.d_edited = mk(self.data), mk(self.mask), mk(self.edited)
        self.counts = torch.zeros(self.L, dtype=torch.int64, device=device)
        self.device = device
        self.K = 0
        self._cap = 0
        self._ev = None
        self.ready = None
        if capacity:
            self._reserve(int(capacity))

    def _reserve(self, cap):
        """ONE packed record buffer (pinned host twin + device): [cap x 4 float64 | cap x int32 | cap x uint32].
        The three arrays the kernels read are views of it, so an upload is one copy and a multi-rank
        broadcast (sharding.broadcast_batch) one collective with nothing to unpack."""
        torch = _torch()
        self._cap = cap
        nbytes = cap * self.RECORD_BYTES
        self._pin = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
        # TWO device copies, written alternately: an upload may run on a side stream while the kernels of the previous
        # batch (which hold raw pointers into the other copy) are still queued or running
        self._bufs = [torch.empty(nbytes, dtype=torch.uint8, device=self.device) for _ in range(2)]
        self._cur = 0
        host = self._pin.numpy()
        self._h_strokes = host[:32 * cap].view(np.float64).reshape(cap, 4)
        self._h_layer = host[32 * cap:36 * cap].view(np.int32)
        self._h_value = host[36 * cap:40 * cap].view(np.uint32)
        self._bind(0)

    def _bind(self, k):
        torch = _torch()
        cap = self._cap
        self._cur = k
        self.packed = self._bufs[k]
        self._d_strokes = self.packed[:32 * cap].view(torch.float64).view(cap, 4)
        self._d_layer = self.packed[32 * cap:36 * cap].view(torch.int32)
        self._d_value = self.packed[36 * cap:40 * cap].view(torch.int32)

    def pack_host(self, strokes, layer_of, values, out):
        """Write one batch in the packed record layout into `out`, a uint8 numpy array of capacity * RECORD_BYTES
        bytes (callers that stage many batches at once, e.g. one table per step of a resident loop)."""
        cap = self._cap
        strokes = np.ascontiguousarray(strokes, dtype=np.float64)
        K = strokes.shape[0]
        dt = _np_dtype_of(self.data[0])
        hs = out[:32 * cap].view(np.float64).reshape(cap, 4)
        hl = out[32 * cap:36 * cap].view(np.int32)
        hv = out[36 * cap:40 * cap].view(np.uint32)
        hs[:K] = strokes
        hs[K:] = np.nan
        hl[:K] = np.asarray(layer_of, dtype=np.int32)
        hl[K:] = 0
        v = np.asarray(values).astype(dt).reshape(K)
        hv[:K] = v.view({1: np.uint8, 2: np.uint16, 4: np.uint32}[dt.itemsize])
        hv[K:] = 0
        return K

    def bind(self, packed, K):
        """Point the batch at a packed record buffer that is already on the device (uint8, capacity * RECORD_BYTES
        bytes, 16-byte aligned): no copy."""
        torch = _torch()
        cap = self._cap
        if packed.numel() != cap * self.RECORD_BYTES or packed.data_ptr() % 8:
            raise TargetMismatch("packed stroke table does not match the batch's capacity")
        self.packed = packed
        self._d_strokes = packed[:32 * cap].view(torch.float64).view(cap, 4)
        self._d_layer = packed[32 * cap:36 * cap].view(torch.int32)
        self._d_value = packed[36 * cap:40 * cap].view(torch.int32)
        return self.use(K)

    def use(self, K):
        """Strokes [0, K) of the packed buffer are the batch (after an upload or a broadcast)."""
        self.K = int(K)
        self.d_strokes, self.d_layer_of, self.d_values = self._d_strokes[:K], self._d_layer[:K], self._d_value[:K]
        return self

    def upload(self, strokes, layer_of, values, fill=False):
        """strokes (K,4) float64 [cx,cy,cz,r]; layer_of (K,) int; values (K,) in plane dtype.  One host->device
        copy from pinned memory.  ``fill``: pad the buffer to its capacity with strokes that can never hit
        (NaN centre and radius) and use all of it -- ranks that receive the buffer by broadcast then need not
        know K (no host read-back on the stroke path)."""
        torch = _torch()
        strokes = np.ascontiguousarray(strokes, dtype=np.float64)
        K = strokes.shape[0]
        dt = _np_dtype_of(self.data[0])
        if K > self._cap or self._cap == 0:                      # (an empty first batch still needs buffers)
            if self._ev is not None:
                self._ev.synchronize()
            self._reserve(max(K, 2 * self._cap, 1))
        if self._ev is not None:
            self._ev.synchronize()            # the previous upload must have left the pinned buffer
        self._h_strokes[:K] = strokes
        self._h_layer[:K] = np.asarray(layer_of, dtype=np.int32)
        v = np.asarray(values).astype(dt).reshape(K)
        self._h_value[:K] = v.view({1: np.uint8, 2: np.uint16, 4: np.uint32}[dt.itemsize])
        if fill:
            self._h_strokes[K:] = np.nan
            self._h_layer[K:] = 0
            self._h_value[K:] = 0
        self._bind(self._cur ^ 1)                 # the copy the queued kernels are NOT reading
        self.packed.copy_(self._pin, non_blocking=True)
        self._ev = torch.cuda.Event()
        self._ev.record()                         # on the current stream: callers that upload on a side stream make the
        #                                           compute stream wait for `ready` before the batch kernel
        self.ready = self._ev
        self.upload_bytes = (self._cap if fill else K) * self.RECORD_BYTES
        return self.use(self._cap if fill else K)


def select_sphere_batch(pos, batch, *, tiles=None):
    """Apply ``batch`` (a StrokeBatch after ``upload``) in ONE pass over the position map.
    Per-layer newly-edited counts accumulate into ``batch.counts`` (device).  ``tiles`` (TileBoxes)
    restricts the pass to the tiles some stroke of the batch can reach."""
    torch = require_cuda()
    n = pos.shape[1] * pos.shape[2]
    for d, m, e in zip(batch.data, batch.mask, batch.edited):
        _check_layer_planes(n, d, m, e)
    if tiles is not None:
        _check(lib().ml_select_sphere_batch_tiles(_ptr(pos), n, int(pos.shape[2]), int(pos.shape[1]),
                                                  _ptr(tiles.boxes), _ptr(tiles.scratch), tiles.nbytes,
                                                  _ptr(batch.d_strokes), _ptr(batch.d_layer_of),
                                                  _ptr(batch.d_values), batch.K, _ptr(batch.d_data),
                                                  _ptr(batch.d_mask), _ptr(batch.d_edited), batch.L, batch.esize,
                                                  _ptr(batch.counts), _stream()))
        return
    _check(lib().ml_select_sphere_batch(_ptr(pos), n, n, _ptr(batch.d_strokes), _ptr(batch.d_layer_of),
                                        _ptr(batch.d_values), batch.K, _ptr(batch.d_data),
                                        _ptr(batch.d_mask), _ptr(batch.d_edited), batch.L, batch.esize,
                                        _ptr(batch.counts), _stream()))


class AttrTiles:
    """[min, max] of a float32 attribute plane per 128 x 4-texel tile plus the tile-list scratch of
    the culled threshold selection.  Valid while the plane's contents do not change."""

    def __init__(self, attr, ranges, scratch, nbytes):
        self.attr_ptr, self.shape = attr.data_ptr(), tuple(attr.shape)
        self.ranges, self.scratch, self.nbytes = ranges, scratch, nbytes


def attr_tiles(attr):
    """Per-tile value ranges of a (rows, width) float32 plane; None when the layout has no tiles
    (width % 128 != 0, unaligned) or the plane is not float32."""
    torch = require_cuda()
    L = lib()
    if attr.dtype != torch.float32 or attr.dim() != 2 or not attr.is_contiguous() or attr.data_ptr() % 16:
        return None
    rows, width = int(attr.shape[0]), int(attr.shape[1])
    nt = int(L.ml_tile_count(width, rows))
    if nt == 0 or (rows * width) % 4:
        return None
    ranges = torch.empty((nt, 2), dtype=torch.float32, device=attr.device)
    _check(L.ml_plane_tile_range(_ptr(attr), width, rows, _ptr(ranges), _stream()))
    nb = int(L.ml_tile_workspace_bytes(width, rows))
    return AttrTiles(attr, ranges, torch.empty(nb, dtype=torch.uint8, device=attr.device), nb)


def select_threshold(attr, valid, lo, hi, data, mask, edited, value, *, counts=None, tiles=None):
    """Attribute-threshold selection: lo <= attr <= hi (closed) where ``valid`` (byte plane or
    None) is non-zero.  Returns newly edited texels.  ``tiles`` (``attr_tiles(attr)``, for planes that
    do not change between selections) restricts the pass to tiles whose value range meets
    [lo, hi]; same planes and count."""
    require_cuda()
    n = attr.numel()
    name = _np_dtype_of(attr).name
    if name not in KIND_CODES or not attr.is_contiguous():
        raise TargetMismatch("unsupported attribute plane (%s)" % name)
    _check_layer_planes(n, data, mask, edited)
    if valid is not None:
        _byte_plane(valid, "valid")
        if valid.numel() != n:
            raise TargetMismatch("valid plane does not match the attribute plane")
    bits, esize = value_bits(value, data)
    ctr = counts if counts is not None else _counters(1, attr.device)
    culled = (tiles is not None and tiles.attr_ptr == attr.data_ptr() and tiles.shape == tuple(attr.shape)
              and all(t.data_ptr() % 16 == 0 for t in (data, mask, edited)) and (valid is None or valid.data_ptr() % 4 == 0))
    if culled:
        _check(lib().ml_select_threshold_tiles(_ptr(attr), _ptr(valid), int(attr.shape[1]), int(attr.shape[0]),
                                               _ptr(tiles.ranges), _ptr(tiles.scratch), tiles.nbytes, float(lo), float(hi),
                                               _ptr(data), esize, bits, _ptr(mask), _ptr(edited), _ptr(ctr), _stream()))
    else:
        _check(lib().ml_select_threshold(_ptr(attr), KIND_CODES[name], _ptr(valid), n, float(lo), float(hi),
                                         _ptr(data), esize, bits, _ptr(mask), _ptr(edited), _ptr(ctr),
                                         _stream()))
    return None if counts is not None else int(ctr[0].item())


def layer_op(op, da, ma, db, mb, dc, mc):
    """(dc, mc) = (da, ma) <op> (db, mb).  Data planes may all be None (mask-only algebra)."""
    require_cuda()
    n = ma.numel()
    if mb.numel() != n or mc.numel() != n:
        raise TargetMismatch("mask planes disagree in size")
    for m in (ma, mb, mc):
        _byte_plane(m, "mask")
    esize = 0
    if dc is not None:
        esize = _np_dtype_of(dc).itemsize
        for d in (da, db):
            if d is not None and (_np_dtype_of(d).itemsize != esize or d.numel() != n or not d.is_contiguous()):
                raise TargetMismatch("data planes disagree in kind or size")
        if da is None or dc.numel() != n or not dc.is_contiguous():
            raise TargetMismatch("data planes disagree in kind or size")
    _check(lib().ml_layer_op(OPS[op] if isinstance(op, str) else int(op), _ptr(da), _ptr(ma), _ptr(db),
                             _ptr(mb), _ptr(dc), _ptr(mc), esize, n, _stream()))


ML_CHAIN_EAGER = 0x100


def layer_chain(datas, masks, ops, dc, mc, *, lazy=True):
    """Fused left-to-right chain ((L0 ops[1] L1) ops[2] L2) ... in one pass.  ``ops[0]`` ignored.
    ``lazy=False`` forces the streaming kernel that reads every data vector (the default reads the
    data of 3..8 one-byte layers only where the masks let it contribute; same result)."""
    require_cuda()
    N = len(masks)
    n = mc.numel()
    esize = 0 if dc is None else _np_dtype_of(dc).itemsize
    for m in list(masks) + [mc]:
        _byte_plane(m, "mask")
        if m.numel() != n:
            raise TargetMismatch("mask planes disagree in size")
    if esize:
        for d in list(datas) + [dc]:
            if _np_dtype_of(d).itemsize != esize or d.numel() != n or not d.is_contiguous():
                raise TargetMismatch("data planes disagree in kind or size")
    dptr = (C.c_void_p * N)(*[(d.data_ptr() if esize else None) for d in (datas if esize else [None] * N)])
    mptr = (C.c_void_p * N)(*[m.data_ptr() for m in masks])
    codes = (C.c_int32 * N)(*[0 if lazy else ML_CHAIN_EAGER] + [OPS[o] if isinstance(o, str) else int(o) for o in list(ops)[1:]])
    _check(lib().ml_layer_chain(N, dptr, mptr, codes, _ptr(dc), _ptr(mc), esize, n, _stream()))


def layer_area(area, masks, *, sums=None, counts=None):
    """Per-layer area: for every mask plane, sum of area over texels with mask != 0 (float64).
    Returns (sums, counts) as numpy arrays, or None when device accumulators are supplied."""
    torch = require_cuda()
    masks = list(masks)
    n = area.numel()
    if area.dtype != torch.float32 or not area.is_contiguous():
        raise TargetMismatch("area must be a contiguous float32 plane")
    for m in masks:
        _byte_plane(m, "mask")
        if m.numel() != n:
            raise TargetMismatch("mask plane does not match the area plane")
    Lc = len(masks)
    own = sums is None
    if own:
        sums = torch.zeros(Lc, dtype=torch.float64, device=area.device)
        counts = torch.zeros(Lc, dtype=torch.int64, device=area.device)
    for l0 in range(0, Lc, 64):
        chunk = masks[l0:l0 + 64]
        mptr = (C.c_void_p * len(chunk))(*[m.data_ptr() for m in chunk])
        _check(lib().ml_layer_area(_ptr(area), mptr, len(chunk), n,
                                   C.c_void_p(sums.data_ptr() + 8 * l0),
                                   None if counts is None else C.c_void_p(counts.data_ptr() + 8 * l0),
                                   _stream()))
    if own:
        return sums.cpu().numpy(), counts.cpu().numpy()
    return None


class PeerRegion:
    """A zeroed cudaMalloc region that other processes of the node can map (CUDA IPC): ``handle`` is the 64-byte
    blob to send them, ``PeerRegion.open(handle)`` maps a peer's region into this process.  ``tensor(dtype)`` views
    the bytes as a torch tensor without copying."""

    def __init__(self, nbytes=None, *, _ptr_value=None, _opened=False):
        require_cuda()
        self.nbytes, self.opened = nbytes, _opened
        if _ptr_value is None:
            p = C.c_void_p()
            _check(lib().ml_peer_alloc(C.byref(p), nbytes))
            self.ptr = p.value
        else:
            self.ptr = _ptr_value

    @property
    def handle(self):
        buf = C.create_string_buffer(64)
        _check(lib().ml_peer_export(self.ptr, buf))
        return buf.raw

    @classmethod
    def open(cls, handle, nbytes):
        p = C.c_void_p()
        _check(lib().ml_peer_open(C.c_char_p(handle), C.byref(p)))
        return cls(nbytes, _ptr_value=p.value, _opened=True)

    def tensor(self, dtype, device):
        torch = _torch()
        item = torch.empty(0, dtype=dtype).element_size()
        typestr = {torch.int64: "<i8", torch.float64: "<f8", torch.uint8: "|u1"}[dtype]

        class _View:
            __cuda_array_interface__ = {"shape": (self.nbytes // item,), "typestr": typestr, "data": (self.ptr, False), "version": 2}
        return torch.as_tensor(_View(), device=device)

    def close(self):
        if self.ptr:
            (lib().ml_peer_close if self.opened else lib().ml_peer_free)(self.ptr)
            self.ptr = None


def layer_area_peers(area, masks, peer_rows, self_index, arrive_table, status, recycle_row=None):
    """Per-layer areas of this rank's slab added straight into EVERY rank's result row over peer memory, followed
    by the signal / wait of the fused reduction (ml_layer_area_peers).  ``peer_rows``: device addresses (ints) of
    the step's row in every rank's region, ``arrive_table``: device int64 tensor holding the addresses of their
    arrival slots, ``status``: device int32[1] raised when the wait times out."""
    torch = require_cuda()
    masks = list(masks)
    n = area.numel()
    if area.dtype != torch.float32 or not area.is_contiguous():
        raise TargetMismatch("area must be a contiguous float32 plane")
    for m in masks:
        _byte_plane(m, "mask")
        if m.numel() != n:
            raise TargetMismatch("mask plane does not match the area plane")
    mptr = (C.c_void_p * len(masks))(*[m.data_ptr() for m in masks])
    rows = (C.c_void_p * len(peer_rows))(*[int(p) for p in peer_rows])
    _check(lib().ml_layer_area_peers(_ptr(area), mptr, len(masks), n, rows, len(peer_rows), int(self_index),
                                     _ptr(arrive_table), _ptr(status), None if recycle_row is None else C.c_void_p(int(recycle_row)),
                                     _stream()))


def label_area(area, data, mask):
    """Area and texel count per label value of a uint8 data plane -> (sums[256], counts[256])."""
    torch = require_cuda()
    n = area.numel()
    if _np_dtype_of(data).itemsize != 1 or data.numel() != n or mask.numel() != n:
        raise TargetMismatch("label_area needs 1-byte data / mask planes matching the area plane")
    sums = torch.zeros(256, dtype=torch.float64, device=area.device)
    counts = torch.zeros(256, dtype=torch.int64, device=area.device)
    _check(lib().ml_label_area(_ptr(area), _ptr(data), _ptr(mask), n, _ptr(sums), _ptr(counts), _stream()))
    return sums.cpu().numpy(), counts.cpu().numpy()


def layer_stats(attr, mask):
    """(count, sum, min, max) of the attribute over mask != 0, float64."""
    torch = require_cuda()
    name = _np_dtype_of(attr).name
    if name not in KIND_CODES or attr.numel() != mask.numel():
        raise TargetMismatch("attribute / mask planes disagree")
    out = torch.tensor([0.0, 0.0, math.inf, -math.inf], dtype=torch.float64, device=attr.device)
    _check(lib().ml_layer_stats(_ptr(attr.contiguous()), KIND_CODES[name], _ptr(_byte_plane(mask, "mask")),
                                attr.numel(), _ptr(out), _stream()))
    c, s, mn, mx = out.tolist()
    return int(c), s, mn, mx


def outline_mask(cov, thickness, *, in_row0=0, out_row0=None, out_rows=None, out=None):
    """SPEC.md:286-289 second pass over a coverage slab (rows [in_row0, in_row0+cov.shape[0]))."""
    torch = require_cuda()
    _byte_plane(cov, "coverage")
    in_rows, w = cov.shape
    out_row0 = in_row0 if out_row0 is None else out_row0
    out_rows = in_rows - (out_row0 - in_row0) if out_rows is None else out_rows
    if out is None:
        out = torch.empty((out_rows, w), dtype=torch.uint8, device=cov.device)
    _check(lib().ml_outline_mask(_ptr(cov), w, in_row0, in_rows, out_row0, out_rows, int(thickness),
                                 _ptr(out), _stream()))
    return out


def apply_padding(outline, edited, radius, data, mask, value, *, in_row0=0, out_row0=None, counts=None,
                  tiles=None, row_range=None):
    """SPEC.md:295-298.  ``edited`` is the input slab (with halo rows), the others output slabs.
    ``tiles``: the TEA stroke's 128 x 8-texel tile bitmap (``tea_texels(..., tiles=...)``); the pass
    then reads only the neighbourhood of the stroke's footprint (same result).  ``row_range`` (culled
    form only) restricts the pass to the output rows [lo, hi) of the slab."""
    require_cuda()
    in_rows, w = edited.shape
    out_rows = outline.shape[0]
    out_row0 = in_row0 if out_row0 is None else out_row0
    _byte_plane(outline, "outline")
    _byte_plane(edited, "edited")
    _check_layer_planes(out_rows * w, data, mask, None)
    bits, esize = value_bits(value, data)
    ctr = counts if counts is not None else _counters(1, edited.device)
    culled = (tiles is not None and in_rows == out_rows and out_row0 == in_row0 and w % 128 == 0 and 0 < radius <= 4
              and all(t.data_ptr() % 16 == 0 for t in (outline, edited, data, mask)))
    if row_range is not None and not culled:
        raise TargetMismatch("row_range needs the tile-culled padding path")
    if culled and row_range is not None:
        _check(lib().ml_apply_padding_tiles_rows(_ptr(outline), _ptr(edited), w, in_rows, int(row_range[0]),
                                                 int(row_range[1]), int(radius), _ptr(tiles), _ptr(data), esize, bits,
                                                 _ptr(mask), _ptr(ctr), _stream()))
    elif culled:
        _check(lib().ml_apply_padding_tiles(_ptr(outline), _ptr(edited), w, in_rows, int(radius), _ptr(tiles),
                                            _ptr(data), esize, bits, _ptr(mask), _ptr(ctr), _stream()))
    else:
        _check(lib().ml_apply_padding(_ptr(outline), _ptr(edited), w, in_row0, in_rows, out_row0, out_rows,
                                      int(radius), _ptr(data), esize, bits, _ptr(mask), _ptr(ctr), _stream()))
    return None if counts is not None else int(ctr[0].item())


def resolve_display(data, mask, lower, upper, positions, colours, out=None):
    """(rows, width, 4) uint8 RGBA plane; mask false -> (0,0,0,0)."""
    torch = require_cuda()
    name = _np_dtype_of(data).name
    if name not in KIND_CODES or data.numel() != mask.numel() or not data.is_contiguous():
        raise TargetMismatch("data / mask planes disagree")
    _byte_plane(mask, "mask")
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    col = np.ascontiguousarray(colours, dtype=np.float64).reshape(-1, 4)
    if out is None:
        out = torch.empty(tuple(mask.shape) + (4,), dtype=torch.uint8, device=data.device)
    _check(lib().ml_resolve_display(_ptr(data), KIND_CODES[name], _ptr(mask), mask.numel(), float(lower), float(upper),
                                    pos.ctypes.data, col.ctypes.data, len(pos), _ptr(out), _stream()))
    return out


def pack_mask(mask):
    """Byte mask plane -> packed bits (MSB first), on the device."""
    torch = require_cuda()
    _byte_plane(mask, "mask")
    n = mask.numel()
    bits = torch.empty((n + 7) // 8, dtype=torch.uint8, device=mask.device)
    _check(lib().ml_pack_mask(_ptr(mask), n, _ptr(bits), _stream()))
    return bits


def unpack_mask(bits, n, out):
    """Packed bits -> 0/1 byte plane ``out`` (n texels), on the device."""
    require_cuda()
    _byte_plane(out, "mask")
    if bits.numel() < (n + 7) // 8 or out.numel() != n:
        raise TargetMismatch("packed mask size mismatch")
    _check(lib().ml_unpack_mask(_ptr(bits), n, _ptr(out), _stream()))
    return out
