"""Shared scene builders for tests (and tests/golden/make_golden.py)."""
import glob
import os

import numpy as np

from paper_2501_14807_b200 import synth
from paper_2501_14807_b200.mesh_core import window_triangles

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def golden_names(prefix):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


def tea_scene_inputs(level, atlas, window, tool_r, tool_xy):
    """Icosphere + chart-grid atlas + default camera + circular tool; everything except the depth
    plane (which the fixture stores, because the reference rendered it)."""
    mesh = synth.icosphere_mesh(int(level))
    cam = synth.default_camera(int(window), int(window))
    win_xy, win_zn = window_triangles(mesh, cam)
    tri_xy = mesh.tri_uv_texels(int(atlas), int(atlas))
    clip = cam.clip_coords(mesh.vertices)[mesh.triangles]
    shape = synth.circle_shape(int(tool_r))
    tw = th = shape.shape[0]
    sfx, sfy = window / (2.0 * tw), window / (2.0 * th)
    bx = 0.5 - (float(tool_xy[0]) - 0.5 * window) / tw
    by = 0.5 - (float(tool_xy[1]) - 0.5 * window) / th
    return dict(mesh=mesh, cam=cam, win_xy=win_xy, win_zn=win_zn, tri_xy=tri_xy, tri_clip=clip,
                shape=shape, sfx=float(sfx), sfy=float(sfy), bx=float(bx), by=float(by))


def terrain_scene_inputs(quads, atlas, window, tool_r):
    """BASELINE config C2's mesh (heightfield, quads x quads cells; 707 -> 999,698 triangles) with the bench
    camera and a circular tool at the window centre: the inputs of the three reference kernels."""
    mesh = synth.heightfield_mesh(int(quads), margin=0.01)
    cam = synth.default_camera(int(window), int(window), eye=(0.5, 0.5, 1.6), target=(0.5, 0.5, 0.0), fovy=40.0,
                               near=0.2, far=5.0)
    win_xy, win_zn = window_triangles(mesh, cam)
    tri_xy = mesh.tri_uv_texels(int(atlas), int(atlas))
    clip = cam.clip_coords(mesh.vertices)[mesh.triangles]
    shape = synth.circle_shape(int(tool_r))
    tw = th = shape.shape[0]
    sfx, sfy = window / (2.0 * tw), window / (2.0 * th)
    return dict(mesh=mesh, cam=cam, win_xy=win_xy, win_zn=win_zn, tri_xy=tri_xy, tri_clip=clip, shape=shape,
                sfx=float(sfx), sfy=float(sfy), bx=0.5, by=0.5)


def eps_of(fix):
    """Fixture eps with the Python type the reference was called with (float vs np.float64)."""
    return np.float64(fix["eps"]) if bool(fix["eps_is_np64"]) else float(fix["eps"])


def random_tea_case(seed, ntri=200, w=64, h=64, plane_dtype=np.uint8, value=7, tri_dtype=np.float64,
                    eps=1e-4):
    """Random TEA stroke inputs (same recipe as the tea_rand_* fixtures)."""
    rng = np.random.default_rng(seed)
    tri = synth.random_soup(rng, ntri, float(max(w, h)), dtype=np.float64)
    tri[..., 1] *= h / float(max(w, h))
    tri = tri.astype(tri_dtype)
    ww, wh = 37.0, 29.0
    clip = np.empty((ntri, 3, 4))
    wc = rng.uniform(0.5, 3.0, size=(ntri, 3))
    wc[rng.random((ntri, 3)) < 0.08] *= -1.0
    clip[..., 3] = wc
    clip[..., 0] = rng.uniform(-1.4, 1.4, size=(ntri, 3)) * np.abs(wc)
    clip[..., 1] = rng.uniform(-1.4, 1.4, size=(ntri, 3)) * np.abs(wc)
    clip[..., 2] = rng.uniform(-1.0, 1.0, size=(ntri, 3)) * np.abs(wc)
    clip = clip.astype(tri_dtype)
    depth = rng.uniform(0.2, 1.0, size=(int(wh), int(ww))).astype(np.float32)
    shape = (rng.random((9, 11)) < 0.7).astype(np.uint8)
    data = rng.integers(0, 5, size=(h, w)).astype(plane_dtype)
    mask = rng.random((h, w)) < 0.1
    edited = (rng.random((h, w)) < 0.05).astype(np.uint8)
    return dict(tri_xy=tri, tri_clip=clip, ww=ww, wh=wh, depth=depth, eps=eps, sfx=1.3, sfy=0.9,
                bx=0.45, by=0.55, shape=shape, data=data, mask=mask, edited=edited, value=value)


def tea_args(c):
    return (c["tri_xy"], c["tri_clip"], c["ww"], c["wh"], c["depth"], c["eps"], c["sfx"], c["sfy"],
            c["bx"], c["by"], c["shape"])


def morton3(x, y, z):
    """Bit interleave, x in bit 0 / y in bit 1 / z in bit 2 of every triple (octant code of KN:267)."""
    def spread(v):
        v = np.asarray(v).astype(np.uint64) & np.uint64(0x1fffff)
        for s, m in ((32, 0x1f00000000ffff), (16, 0x1f0000ff0000ff), (8, 0x100f00f00f00f00f),
                     (4, 0x10c30c30c30c30c3), (2, 0x1249249249249249)):
            v = (v | (v << np.uint64(s))) & np.uint64(m)
        return v
    return spread(x) | (spread(y) << np.uint64(1)) | (spread(z) << np.uint64(2))


def bounding_cube(verts, pad=1e-3):
    """Root cube of SPEC:333: the bounding box cubified to its largest extent (slightly padded)."""
    lo, hi = verts.min(0), verts.max(0)
    side = float((hi - lo).max()) * (1.0 + pad)
    centre = 0.5 * (lo + hi)
    return (centre - 0.5 * side).astype(np.float64), side


def build_leaf_grid(expand, verts, tris, cube_min, side, depth, coarse_bits=2):
    """Level-by-level surface octree built with ``expand`` (any implementation of
    KN:303 ``expand_pairs_ordered``); returns the leaf arrays ``raycast`` (KN:361) consumes and the
    per-level (cells, tri) lists for comparing implementations."""
    T = tris.shape[0]
    parent_cells = np.zeros((1, 3), np.uint32)
    pair_parent = np.zeros(T, np.int64)
    pair_tri = np.arange(T, dtype=np.int32)
    levels = []
    cells = np.zeros((T, 3), np.uint32)
    for lvl in range(1, depth + 1):
        child_h = side / float(1 << lvl)
        cells, pair_tri = expand(verts, tris, parent_cells, pair_parent, pair_tri, cube_min, child_h)
        levels.append((cells, pair_tri))
        key = morton3(cells[:, 0], cells[:, 1], cells[:, 2])
        ukeys, first, inv = np.unique(key, return_index=True, return_inverse=True)
        parent_cells, pair_parent = cells[first], inv.astype(np.int64)
    key = morton3(cells[:, 0], cells[:, 1], cells[:, 2])
    order = np.lexsort((pair_tri, key))
    keys, counts = np.unique(key[order], return_counts=True)
    offsets = np.zeros(keys.shape[0] + 1, np.int64)
    offsets[1:] = np.cumsum(counts)
    n_cells = 1 << depth
    cb = min(coarse_bits, depth)
    shift = depth - cb
    coarse = np.zeros((1 << cb,) * 3, np.uint8)
    coarse[cells[:, 0] >> shift, cells[:, 1] >> shift, cells[:, 2] >> shift] = 1
    return dict(keys=keys.astype(np.uint64), offsets=offsets, tri_idx=pair_tri[order].astype(np.int32),
                h=side / float(n_cells), n_cells=n_cells, coarse=coarse, coarse_shift=shift,
                levels=levels)


def camera_rays(cam, pixels):
    """World-space rays through window pixel centres (origin = eye), float64; ``pixels`` (N,2)."""
    inv = np.linalg.inv(np.asarray(cam.mvp, np.float64))
    px = (np.asarray(pixels, np.float64) + 0.5)
    ndc = np.stack([px[:, 0] / cam.width * 2.0 - 1.0, px[:, 1] / cam.height * 2.0 - 1.0], 1)
    near = np.concatenate([ndc, -np.ones((len(px), 1)), np.ones((len(px), 1))], 1) @ inv.T
    far = np.concatenate([ndc, np.ones((len(px), 1)), np.ones((len(px), 1))], 1) @ inv.T
    near, far = near[:, :3] / near[:, 3:], far[:, :3] / far[:, 3:]
    d = far - near
    return np.ascontiguousarray(near), np.ascontiguousarray(d / np.linalg.norm(d, axis=1, keepdims=True))


def brute_raycast(origins, dirs, verts, tris):
    """Per-ray nearest hit over ALL triangles with the reference's Moeller-Trumbore expression order
    (numpy, vectorised over triangles): the brute-force oracle of SPEC.md:358, 380."""
    v0, v1, v2 = verts[tris[:, 0]], verts[tris[:, 1]], verts[tris[:, 2]]
    e1, e2 = v1 - v0, v2 - v0
    best_t = np.full(len(origins), np.inf)
    best_tri = np.full(len(origins), -1, np.int64)
    for i, (o, u) in enumerate(zip(origins, dirs)):
        px = u[1] * e2[:, 2] - u[2] * e2[:, 1]
        py = u[2] * e2[:, 0] - u[0] * e2[:, 2]
        pz = u[0] * e2[:, 1] - u[1] * e2[:, 0]
        det = e1[:, 0] * px + e1[:, 1] * py + e1[:, 2] * pz
        ok = det != 0.0
        inv = 1.0 / np.where(ok, det, 1.0)
        tv = o - v0
        bu = (tv[:, 0] * px + tv[:, 1] * py + tv[:, 2] * pz) * inv
        ok &= (bu >= 0.0) & (bu <= 1.0)
        qx = tv[:, 1] * e1[:, 2] - tv[:, 2] * e1[:, 1]
        qy = tv[:, 2] * e1[:, 0] - tv[:, 0] * e1[:, 2]
        qz = tv[:, 0] * e1[:, 1] - tv[:, 1] * e1[:, 0]
        bv = (u[0] * qx + u[1] * qy + u[2] * qz) * inv
        ok &= (bv >= 0.0) & (bu + bv <= 1.0)
        t = (e2[:, 0] * qx + e2[:, 1] * qy + e2[:, 2] * qz) * inv
        ok &= t >= 0.0
        t = np.where(ok, t, np.inf)
        j = int(np.argmin(t))                                         # first minimum = smallest index
        if np.isfinite(t[j]):
            best_t[i], best_tri[i] = t[j], j
    return best_t, best_tri


def octree_rays(window, seed, nrandom):
    """Camera rays of a window x window view of the unit sphere plus seeded random rays (axis-parallel,
    integer-direction and interior-origin cases included); float64 (N,3) origins and directions."""
    rng = np.random.default_rng(seed)
    cam = synth.default_camera(int(window), int(window), eye=(0.4, 0.3, 3.2))
    ys, xs = np.mgrid[0:window, 0:window]
    o, d = camera_rays(cam, np.stack([xs.ravel(), ys.ravel()], 1))
    ro = rng.uniform(-1.5, 1.5, size=(nrandom, 3))
    rd = rng.normal(size=(nrandom, 3))
    rd[: nrandom // 8, 1] = 0.0
    rd[nrandom // 8: nrandom // 4] = np.round(rd[nrandom // 8: nrandom // 4])
    ro[nrandom // 2:] *= 0.3                                              # origins inside the sphere
    return np.concatenate([o, ro]), np.concatenate([d, rd])


def c1_stroke_script(window):
    """Eight strokes of a session on config C1: positions, radii, values and the tool bitmaps' kind."""
    rng = np.random.default_rng(81)
    out = []
    for k in range(8):
        r = int(rng.integers(4, 60))
        out.append(dict(px=float(rng.uniform(0.2, 0.8) * window), py=float(rng.uniform(0.2, 0.8) * window), r=r,
                        square=bool(k % 3 == 2), value=int(rng.integers(1, 250))))
    return out


def stroke_tool_map(st, window):
    """Tool bitmap and the kernel's (sfx, sfy, bx, by) of one scripted stroke (KN:187-188 via SPEC:259-267)."""
    shape = synth.square_shape(2 * st["r"] + 1) if st["square"] else synth.circle_shape(st["r"])
    th, tw = shape.shape
    return shape, (window / (2.0 * tw), window / (2.0 * th), 0.5 - (st["px"] - 0.5 * window) / tw,
                   0.5 - (st["py"] - 0.5 * window) / th)
