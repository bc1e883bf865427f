"""Generate tests/golden/*.npz by running the REFERENCE's own numpy kernels.

Run in the build container only (needs /root/reference, which does not exist on the GPU box):

    python tests/golden/make_golden.py

Each fixture stores the seeded inputs and the planes / counts the reference produced, so the
oracle (oracle/kn_port.c) and the CUDA library can be pinned against the reference without the
reference being present.  Scenes deliberately mix float32 / float64 inputs, both windings,
vertices snapped onto texel centres and corners (tie rule), degenerate triangles, pre-dirtied
planes, all plane kinds and both eps promotion modes.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from meshlayers import _kernels_numpy as KN  # noqa: E402  (the reference itself)

from paper_2501_14807_b200 import synth  # noqa: E402
sys.path.insert(0, os.path.dirname(HERE))
import helpers  # noqa: E402  (tests/helpers.py)


def soup(rng, ntri, w, h, dtype):
    tri = synth.random_soup(rng, ntri, float(max(w, h)), dtype=np.float64)
    tri[..., 1] *= h / float(max(w, h))
    return tri.astype(dtype)


def gen_coverage(seed, ntri, w, h, dtype, dirty):
    rng = np.random.default_rng(seed)
    tri = soup(rng, ntri, w, h, dtype)
    out0 = np.zeros((h, w), np.uint8)
    if dirty:
        out0[rng.random((h, w)) < 0.05] = 1
        out0[rng.random((h, w)) < 0.02] = 7          # non-{0,1} bytes must become exactly 1
    out = out0.copy()
    written = KN.coverage_fill(tri, w, h, out)
    return dict(tri_xy=tri, width=w, height=h, out0=out0, out=out, written=written)


def gen_depth(seed, ntri, w, h, dtype):
    rng = np.random.default_rng(seed)
    tri = soup(rng, ntri, w, h, dtype)
    zn = rng.uniform(-1.3, 1.1, size=(ntri, 3)).astype(dtype)
    d0 = np.ones((h, w), np.float32)
    d0[rng.random((h, w)) < 0.1] = np.float32(0.4)
    depth = d0.copy()
    KN.raster_depth(tri, zn, depth)                  # count is order dependent: not stored
    return dict(tri_xy=tri, tri_zn=zn, depth0=d0, depth=depth)


def gen_tea_random(seed, ntri, w, h, dtype, plane_dtype, eps, value):
    rng = np.random.default_rng(seed)
    tri = soup(rng, ntri, w, h, dtype)
    ww, wh = 37.0, 29.0
    clip = np.empty((ntri, 3, 4))
    wc = rng.uniform(0.5, 3.0, size=(ntri, 3))
    wc[rng.random((ntri, 3)) < 0.08] *= -1.0         # some vertices behind the projector
    clip[..., 3] = wc
    clip[..., 0] = rng.uniform(-1.4, 1.4, size=(ntri, 3)) * np.abs(wc)
    clip[..., 1] = rng.uniform(-1.4, 1.4, size=(ntri, 3)) * np.abs(wc)
    clip[..., 2] = rng.uniform(-1.0, 1.0, size=(ntri, 3)) * np.abs(wc)
    clip = clip.astype(dtype)
    depth = rng.uniform(0.2, 1.0, size=(int(wh), int(ww))).astype(np.float32)
    th, tw = 9, 11
    shape = (rng.random((th, tw)) < 0.7).astype(np.uint8)
    sfx, sfy, bx, by = 1.3, 0.9, 0.45, 0.55
    data0 = (rng.integers(0, 5, size=(h, w))).astype(plane_dtype)
    mask0 = (rng.random((h, w)) < 0.1)
    edited0 = (rng.random((h, w)) < 0.05).astype(np.uint8)
    data, mask, edited = data0.copy(), mask0.copy(), edited0.copy()
    ec, fr = KN.raster_tea(tri, clip, ww, wh, depth, eps, sfx, sfy, bx, by, shape, data, mask, edited, value)
    return dict(tri_xy=tri, tri_clip=clip, ww=ww, wh=wh, depth=depth, eps=np.float64(eps),
                eps_is_np64=isinstance(eps, np.float64), sfx=sfx, sfy=sfy, bx=bx, by=by, shape=shape,
                data0=data0, mask0=mask0, edited0=edited0, data=data, mask=mask, edited=edited,
                value=np.array(value, dtype=plane_dtype), edited_count=ec, fragments=fr)


def gen_tea_scene(level, atlas, window, tool_r, tool_xy, eps):
    """Icosphere + chart-grid atlas + perspective camera + circular tool (small)."""
    s = helpers.tea_scene_inputs(level, atlas, window, tool_r, tool_xy)
    depth = np.ones((window, window), np.float32)
    KN.raster_depth(s["win_xy"], s["win_zn"], depth)
    data = np.zeros((atlas, atlas), np.uint8)
    mask = np.zeros((atlas, atlas), bool)
    edited = np.zeros((atlas, atlas), bool)
    ec, fr = KN.raster_tea(s["tri_xy"], s["tri_clip"], float(window), float(window), depth, eps,
                           s["sfx"], s["sfy"], s["bx"], s["by"], s["shape"], data, mask, edited, 7)
    return dict(level=level, atlas=atlas, window=window, tool_r=tool_r, tool_xy=np.array(tool_xy, float),
                eps=np.float64(eps), eps_is_np64=False, depth=depth, data=np.packbits(data != 0),
                data_value=7, mask=np.packbits(mask), edited=np.packbits(edited),
                edited_count=ec, fragments=fr,
                cov_count=int(_coverage_count(s["tri_xy"], atlas)))


def _coverage_count(tri_xy, atlas):
    out = np.zeros((atlas, atlas), np.uint8)
    return KN.coverage_fill(tri_xy, atlas, atlas, out)


def gen_expand(seed, ntri, npar, npair, dtype, snap):
    """expand_pairs_ordered (KN:303) on random (parent cell, triangle) pairs; ``snap`` puts vertices
    on cell faces / corners so the closed-box (touching counts) rule of KN:213-214 is exercised."""
    rng = np.random.default_rng(seed)
    level = 3
    child_h = 1.0 / (1 << (level + 1))
    cube_min = np.array([-0.5, -0.25, 0.125])
    parent_cells = rng.integers(0, 1 << level, size=(npar, 3)).astype(np.uint32)
    ctr = cube_min + (rng.integers(0, 1 << level, size=(ntri, 1, 3)) + 0.5) * (2.0 * child_h)
    pts = ctr + rng.normal(0.0, 1.5 * child_h, size=(ntri, 3, 3))
    if snap:
        m = rng.random(pts.shape) < 0.5
        pts[m] = (cube_min + np.round((pts - cube_min) / child_h) * child_h)[m]
    verts = pts.reshape(-1, 3).astype(dtype)
    tris = np.arange(3 * ntri, dtype=np.int64).reshape(ntri, 3)
    dup = rng.random(ntri) < 0.1
    tris[dup, 2] = tris[dup, 0]                                     # degenerate (segment) triangles
    pair_tri = rng.integers(0, ntri, size=npair).astype(np.int32)
    # parents near their triangle so that a good share of the octants is hit
    want = np.clip(np.floor((pts[pair_tri].mean(1) - cube_min) / (2.0 * child_h)), 0, (1 << level) - 1)
    far = rng.random(npair) < 0.3
    pair_parent = np.empty(npair, np.int64)
    for i in range(npair):
        if far[i]:
            pair_parent[i] = rng.integers(0, npar)
        else:
            d = np.abs(parent_cells.astype(np.int64) - want[i].astype(np.int64)).sum(1)
            pair_parent[i] = int(np.argmin(d))
    cells, tri = KN.expand_pairs_ordered(verts, tris, parent_cells, pair_parent, pair_tri, cube_min, child_h)
    return dict(verts=verts, tris=tris, parent_cells=parent_cells, pair_parent=pair_parent,
                pair_tri=pair_tri, cube_min=cube_min, child_h=np.float64(child_h), cells=cells, tri=tri)


def gen_octree_scene(level, depth, window, coarse_bits, seed, nrandom):
    """Surface octree of an icosphere built with the REFERENCE's expand_pairs_ordered, then the
    reference's raycast (KN:361) for a window of camera rays plus random / axis-parallel / outside /
    zero-direction rays.  The per-level expansion inputs and outputs are stored too."""
    rng = np.random.default_rng(seed)
    mesh = synth.icosphere_mesh(int(level))
    verts = np.ascontiguousarray(mesh.vertices, np.float64)
    tris = np.ascontiguousarray(mesh.triangles, np.int64)
    cube_min, side = helpers.bounding_cube(verts)
    g = helpers.build_leaf_grid(KN.expand_pairs_ordered, verts, tris, cube_min, side, depth, coarse_bits)
    cam = synth.default_camera(window, window)
    ys, xs = np.mgrid[0:window, 0:window]
    o, d = helpers.camera_rays(cam, np.stack([xs.ravel(), ys.ravel()], 1))
    ro = rng.uniform(-1.6, 1.6, size=(nrandom, 3))
    rd = rng.normal(size=(nrandom, 3))
    rd[: nrandom // 4, rng.integers(0, 3)] = 0.0                    # axis-parallel slabs (KN:393-396)
    rd[nrandom // 4: nrandom // 3] = np.round(rd[nrandom // 4: nrandom // 3])   # ties between t_max axes
    rd[-3:] = 0.0                                                   # zero direction: marches in place
    ro[-2] = 0.0
    ro[-1] = (0.2, -0.1, 0.95)
    origins = np.concatenate([o, ro])
    dirs = np.concatenate([d, rd])
    best_t, best_tri, leaf = KN.raycast(origins, dirs, g["keys"], g["offsets"], g["tri_idx"], verts, tris,
                                        cube_min, g["h"], g["n_cells"], g["coarse"], g["coarse_shift"],
                                        helpers.morton3)
    nc_t, nc_tri, nc_leaf = KN.raycast(origins, dirs, g["keys"], g["offsets"], g["tri_idx"], verts, tris,
                                       cube_min, g["h"], g["n_cells"], None, 0, helpers.morton3)
    assert np.array_equal(nc_t, best_t) and np.array_equal(nc_tri, best_tri) and np.array_equal(nc_leaf, leaf)
    out = dict(level=level, depth=depth, cube_min=cube_min, side=np.float64(side), origins=origins, dirs=dirs,
               keys=g["keys"], offsets=g["offsets"], tri_idx=g["tri_idx"], h=np.float64(g["h"]),
               n_cells=g["n_cells"], coarse=g["coarse"], coarse_shift=g["coarse_shift"],
               best_t=best_t, best_tri=best_tri, leaf_pos=leaf)
    for i, (c, t) in enumerate(g["levels"]):
        out["level%d_cells" % (i + 1)] = c
        out["level%d_tri" % (i + 1)] = t
    return out


def gen_c1_digests():
    """BASELINE config C1 at full size through the REFERENCE: the planes are 1 MB each, so the fixture
    stores their SHA-256 digests and the counts; the inputs are rebuilt from helpers.tea_scene_inputs."""
    import hashlib
    A, W, r = 1024, 512, 40
    s = helpers.tea_scene_inputs(5, A, W, r, (W / 2.0, W / 2.0))
    dig = lambda a: np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), np.uint8)  # noqa: E731
    cov = np.zeros((A, A), np.uint8)
    written = KN.coverage_fill(s["tri_xy"], A, A, cov)
    depth = np.ones((W, W), np.float32)
    KN.raster_depth(s["win_xy"], s["win_zn"], depth)
    data, mask, edited = np.zeros((A, A), np.uint8), np.zeros((A, A), bool), np.zeros((A, A), bool)
    ec, fr = KN.raster_tea(s["tri_xy"], s["tri_clip"], float(W), float(W), depth, 1e-4, s["sfx"], s["sfy"], s["bx"],
                           s["by"], s["shape"], data, mask, edited, 7)
    return dict(level=5, atlas=A, window=W, tool_r=r, tool_xy=np.array([W / 2.0, W / 2.0]), eps=1e-4, value=7,
                written=written, edited_count=ec, fragments=fr, cov_sha=dig(cov), depth_sha=dig(depth),
                data_sha=dig(data), mask_sha=dig(mask.view(np.uint8)), edited_sha=dig(edited.view(np.uint8)))


def gen_c2_digests():
    """BASELINE config C2's mesh (999,698 triangles) at a 4096^2 atlas through the REFERENCE -- about ten
    minutes of numpy per-triangle loops, so it only runs with `make_golden.py --c2`."""
    import hashlib
    import time
    Q, A, W, r = 707, 4096, 1024, 70
    s = helpers.terrain_scene_inputs(Q, A, W, r)
    dig = lambda a: np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), np.uint8)  # noqa: E731
    t0 = time.time()
    cov = np.zeros((A, A), np.uint8)
    written = KN.coverage_fill(s["tri_xy"], A, A, cov)
    print("coverage", written, time.time() - t0, flush=True)
    depth = np.ones((W, W), np.float32)
    KN.raster_depth(s["win_xy"], s["win_zn"], depth)
    print("depth", time.time() - t0, flush=True)
    data, mask, edited = np.zeros((A, A), np.uint8), np.zeros((A, A), bool), np.zeros((A, A), bool)
    ec, fr = KN.raster_tea(s["tri_xy"], s["tri_clip"], float(W), float(W), depth, 1e-4, s["sfx"], s["sfy"], s["bx"],
                           s["by"], s["shape"], data, mask, edited, 7)
    print("tea", ec, fr, time.time() - t0, flush=True)
    return dict(quads=Q, atlas=A, window=W, tool_r=r, eps=1e-4, value=7, triangles=s["mesh"].num_triangles,
                written=written, edited_count=ec, fragments=fr, cov_sha=dig(cov), depth_sha=dig(depth),
                data_sha=dig(data), mask_sha=dig(mask.view(np.uint8)), edited_sha=dig(edited.view(np.uint8)),
                reference_seconds=time.time() - t0)


def gen_octree_digests():
    """A larger octree scene through the REFERENCE (icosphere level 5 = 20,480 triangles, depth 8, 16k camera
    rays + 4k random rays): digests of the leaf arrays and of the ray-cast results; inputs are rebuilt from
    seeds by the tests."""
    import hashlib
    dig = lambda a: np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), np.uint8)  # noqa: E731
    level, depth, window, cb, seed, nrandom = 5, 8, 128, 4, 63, 4096
    mesh = synth.icosphere_mesh(level)
    verts = np.ascontiguousarray(mesh.vertices, np.float64)
    tris = np.ascontiguousarray(mesh.triangles, np.int64)
    cube_min, side = helpers.bounding_cube(verts)
    g = helpers.build_leaf_grid(KN.expand_pairs_ordered, verts, tris, cube_min, side, depth, cb)
    origins, dirs = helpers.octree_rays(window, seed, nrandom)
    bt, btri, leaf = KN.raycast(origins, dirs, g["keys"], g["offsets"], g["tri_idx"], verts, tris, cube_min, g["h"],
                                g["n_cells"], g["coarse"], g["coarse_shift"], helpers.morton3)
    return dict(level=level, depth=depth, window=window, coarse_bits=cb, seed=seed, nrandom=nrandom,
                leaves=g["keys"].shape[0], rows=g["tri_idx"].shape[0], hits=int(np.isfinite(bt).sum()),
                keys_sha=dig(g["keys"]), offsets_sha=dig(g["offsets"]), tri_idx_sha=dig(g["tri_idx"]),
                level_rows=np.array([len(t) for _, t in g["levels"]]),
                best_t_sha=dig(bt), best_tri_sha=dig(btri.astype(np.int32)), leaf_sha=dig(leaf.astype(np.int64)))


def gen_c1_session_digests():
    """A session of eight strokes on config C1 through the REFERENCE (the layer planes accumulate, the edited
    mask is fresh per stroke): counts per stroke and digests of the planes after every stroke."""
    import hashlib
    A, W = 1024, 512
    s = helpers.tea_scene_inputs(5, A, W, 10, (W / 2.0, W / 2.0))
    dig = lambda a: np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), np.uint8)  # noqa: E731
    depth = np.ones((W, W), np.float32)
    KN.raster_depth(s["win_xy"], s["win_zn"], depth)
    data, mask = np.zeros((A, A), np.uint8), np.zeros((A, A), bool)
    counts, dsha, msha, esha = [], [], [], []
    for st in helpers.c1_stroke_script(W):
        shape = synth.square_shape(2 * st["r"] + 1) if st["square"] else synth.circle_shape(st["r"])
        th, tw = shape.shape
        sfx, sfy = W / (2.0 * tw), W / (2.0 * th)
        bx, by = 0.5 - (st["px"] - 0.5 * W) / tw, 0.5 - (st["py"] - 0.5 * W) / th
        edited = np.zeros((A, A), bool)
        counts.append(KN.raster_tea(s["tri_xy"], s["tri_clip"], float(W), float(W), depth, 1e-4, sfx, sfy, bx, by,
                                    shape, data, mask, edited, st["value"]))
        dsha.append(dig(data)); msha.append(dig(mask.view(np.uint8))); esha.append(dig(edited.view(np.uint8)))
    return dict(atlas=A, window=W, counts=np.array(counts, np.int64), data_sha=np.stack(dsha), mask_sha=np.stack(msha),
                edited_sha=np.stack(esha))


def main():
    if "--session" in sys.argv:
        d = gen_c1_session_digests()
        np.savez_compressed(os.path.join(HERE, "c1_session_digests.npz"), **d)
        print(d["counts"])
        return
    if "--octree" in sys.argv:
        d = gen_octree_digests()
        np.savez_compressed(os.path.join(HERE, "octree_digests.npz"), **d)
        print({k: v for k, v in d.items() if not k.endswith("_sha")})
        return
    if "--c2" in sys.argv:
        d = gen_c2_digests()
        np.savez_compressed(os.path.join(HERE, "c2_digests.npz"), **d)
        return
    out = {}
    out["c1_digests"] = gen_c1_digests()
    out["octree_expand_a"] = gen_expand(51, 60, 40, 400, np.float64, snap=False)
    out["octree_expand_snap"] = gen_expand(52, 60, 40, 400, np.float64, snap=True)
    out["octree_expand_f32"] = gen_expand(53, 50, 30, 300, np.float32, snap=True)
    out["octree_scene_d4"] = gen_octree_scene(2, 4, 24, 2, 61, 120)
    out["octree_scene_d6"] = gen_octree_scene(3, 6, 32, 3, 62, 160)
    out["coverage_a"] = gen_coverage(11, 160, 48, 40, np.float64, dirty=False)
    out["coverage_b"] = gen_coverage(12, 160, 33, 57, np.float32, dirty=True)
    out["coverage_big"] = gen_coverage(13, 12, 96, 96, np.float64, dirty=False)
    out["depth_a"] = gen_depth(21, 140, 40, 36, np.float64)
    out["depth_b"] = gen_depth(22, 140, 31, 45, np.float32)
    kinds = [(np.uint8, 7), (np.int16, -1234), (np.float32, 2.5), (np.uint32, 4000000000),
             (np.float16, 0.333), (np.int8, -3), (np.int32, -70000)]
    for k, (dt, val) in enumerate(kinds):
        eps = 1e-4 if k % 2 == 0 else np.float64(1e-4)
        out["tea_rand_%d" % k] = gen_tea_random(31 + k, 150, 44, 38, np.float64 if k % 3 else np.float32,
                                                dt, eps, val)
    out["tea_scene_centre"] = gen_tea_scene(2, 128, 96, 12, (48.0, 48.0), 1e-4)
    out["tea_scene_edge"] = gen_tea_scene(2, 128, 96, 20, (80.0, 30.0), 1e-4)
    out["tea_scene_background"] = gen_tea_scene(1, 64, 64, 4, (3.0, 3.0), 1e-4)
    # eps promotion (KN:185): Python-float eps is added in float32, np.float64 eps in float64
    tri = np.array([[[-10.0, -10.0], [30.0, -10.0], [-10.0, 30.0]]])
    dv, eps = np.float32(0.6), 1e-9
    clip = np.zeros((1, 3, 4))
    clip[..., 3] = 1.0
    clip[..., 2] = (float(dv) + 0.5 * eps) * 2.0 - 1.0
    counts = []
    for e in (eps, np.float64(eps)):
        data, mask, edited = np.zeros((4, 4), np.uint8), np.zeros((4, 4), bool), np.zeros((4, 4), bool)
        counts.append(KN.raster_tea(tri, clip, 4.0, 4.0, np.full((4, 4), dv, np.float32), e, 0.5, 0.5, 0.5,
                                    0.5, np.ones((1, 1), np.uint8), data, mask, edited, 1)[0])
    out["epsmode"] = dict(tri_xy=tri, tri_clip=clip, depth_value=dv, eps=np.float64(eps),
                          edited_weak=counts[0], edited_f64=counts[1])
    for name, d in out.items():
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)
        print(name, {k: (v.shape if hasattr(v, "shape") and getattr(v, "ndim", 0) else v) for k, v in d.items()
                     if k in ("written", "edited_count", "fragments", "cov_count")},
              {k: v.shape for k, v in d.items() if k in ("cells", "keys", "best_t")})


if __name__ == "__main__":
    main()
