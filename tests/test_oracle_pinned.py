"""Pin the oracle (oracle/kn_port.c) against the reference's own outputs (tests/golden/*.npz,
made by tests/golden/make_golden.py from /root/reference) and the SPEC known-answer tests.
CPU only."""
import numpy as np
import pytest

import helpers
from oracle import kn


# ------------------------------------------------------------------ golden vectors (reference outputs)

@pytest.mark.parametrize("name", helpers.golden_names("coverage_"))
@pytest.mark.parametrize("threads", [0, 3])
def test_coverage_matches_reference(name, threads):
    g = helpers.golden(name)
    out = g["out0"].copy()
    written = kn.coverage_fill(g["tri_xy"], int(g["width"]), int(g["height"]), out, threads=threads)
    assert np.array_equal(out, g["out"])
    assert written == int(g["written"])


@pytest.mark.parametrize("name", helpers.golden_names("depth_"))
@pytest.mark.parametrize("threads", [0, 3])
def test_depth_matches_reference(name, threads):
    g = helpers.golden(name)
    depth = g["depth0"].copy()
    kn.raster_depth(g["tri_xy"], g["tri_zn"], depth, threads=threads)
    assert np.array_equal(depth.view(np.uint32), g["depth"].view(np.uint32))


@pytest.mark.parametrize("name", helpers.golden_names("tea_rand_"))
@pytest.mark.parametrize("threads", [0, 3])
def test_tea_random_matches_reference(name, threads):
    g = helpers.golden(name)
    data, mask, edited = g["data0"].copy(), g["mask0"].copy(), g["edited0"].copy()
    ec, fr = kn.raster_tea(g["tri_xy"], g["tri_clip"], float(g["ww"]), float(g["wh"]), g["depth"],
                           helpers.eps_of(g), float(g["sfx"]), float(g["sfy"]), float(g["bx"]), float(g["by"]),
                           g["shape"], data, mask, edited, g["value"][()], threads=threads)
    assert (ec, fr) == (int(g["edited_count"]), int(g["fragments"]))
    assert np.array_equal(data.view(np.uint8), g["data"].view(np.uint8))
    assert np.array_equal(mask, g["mask"])
    assert np.array_equal(edited, g["edited"])


@pytest.mark.parametrize("name", helpers.golden_names("tea_scene_"))
def test_tea_scene_matches_reference(name):
    g = helpers.golden(name)
    s = helpers.tea_scene_inputs(g["level"], g["atlas"], g["window"], g["tool_r"], g["tool_xy"])
    A, W = int(g["atlas"]), int(g["window"])
    depth = np.ones((W, W), np.float32)
    kn.raster_depth(s["win_xy"], s["win_zn"], depth)
    assert np.array_equal(depth.view(np.uint32), g["depth"].view(np.uint32))
    data = np.zeros((A, A), np.uint8)
    mask = np.zeros((A, A), bool)
    edited = np.zeros((A, A), bool)
    ec, fr = kn.raster_tea(s["tri_xy"], s["tri_clip"], float(W), float(W), depth, helpers.eps_of(g),
                           s["sfx"], s["sfy"], s["bx"], s["by"], s["shape"], data, mask, edited, 7)
    assert (ec, fr) == (int(g["edited_count"]), int(g["fragments"]))
    assert np.array_equal(np.packbits(mask), g["mask"])
    assert np.array_equal(np.packbits(edited), g["edited"])
    assert np.array_equal(np.packbits(data != 0), g["data"])
    assert set(np.unique(data)) <= {0, 7}
    cov = np.zeros((A, A), np.uint8)
    assert kn.coverage_fill(s["tri_xy"], A, A, cov) == int(g["cov_count"])


def _epsmode_counts(fn):
    g = helpers.golden("epsmode")
    res = []
    for e in (float(g["eps"]), np.float64(g["eps"])):
        data, mask, edited = np.zeros((4, 4), np.uint8), np.zeros((4, 4), bool), np.zeros((4, 4), bool)
        depth = np.full((4, 4), g["depth_value"], np.float32)
        res.append(fn(g["tri_xy"], g["tri_clip"], 4.0, 4.0, depth, e, 0.5, 0.5, 0.5, 0.5,
                      np.ones((1, 1), np.uint8), data, mask, edited, 1)[0])
    return res, [int(g["edited_weak"]), int(g["edited_f64"])]


def test_eps_promotion_mode_matches_reference():
    """KN:185: float32(depth)+eps is rounded to float32 for a Python-float eps but stays float64
    for a np.float64 eps; the fixture holds what the reference returned in both modes."""
    got, want = _epsmode_counts(kn.raster_tea)
    assert got == want == [0, 16]


# ------------------------------------------------------------------ SPEC known answers

def _square(x0, y0, s):
    return np.array([[[x0, y0], [x0 + s, y0], [x0 + s, y0 + s]],
                     [[x0, y0], [x0 + s, y0 + s], [x0, y0 + s]]], dtype=np.float64)


def test_spec_10x10_square_covers_100_cells():
    out = np.zeros((64, 64), np.uint8)
    assert kn.coverage_fill(_square(20.0, 30.0, 10.0), 64, 64, out) == 100
    assert out[30:40, 20:30].all() and out.sum() == 100


def test_spec_coverage_winding_and_permutation_invariant():
    tri = _square(20.0, 30.0, 10.0)
    ref = np.zeros((64, 64), np.uint8)
    kn.coverage_fill(tri, 64, 64, ref)
    for perm in ([0, 2, 1], [1, 2, 0], [2, 1, 0]):
        out = np.zeros((64, 64), np.uint8)
        assert kn.coverage_fill(tri[::-1, perm], 64, 64, out) == 100
        assert np.array_equal(out, ref)


def test_spec_two_triangles_tile_unit_square():
    out = np.zeros((64, 64), np.uint8)
    assert kn.coverage_fill(_square(0.0, 0.0, 64.0), 64, 64, out) == 4096


def test_spec_triangle_covering_three_centres():
    tri = np.array([[[1.2, 1.2], [3.4, 1.2], [1.2, 3.4]]])
    out = np.zeros((6, 6), np.uint8)
    kn.coverage_fill(tri, 6, 6, out)
    ys, xs = np.nonzero(out)
    assert sorted(zip(xs.tolist(), ys.tolist())) == [(1, 1), (1, 2), (2, 1)]


def test_spec_watertight_quad_split():                     # SPEC.md:141; KN:13-15
    quad = _square(2.5, 2.5, 8.0)                          # diagonal passes through texel centres
    a = np.zeros((16, 16), np.uint8)
    b = np.zeros((16, 16), np.uint8)
    na = kn.coverage_fill(quad[:1], 16, 16, a)
    nb = kn.coverage_fill(quad[1:], 16, 16, b)
    assert not (a & b).any()                               # no texel owned twice
    both = np.zeros((16, 16), np.uint8)
    assert kn.coverage_fill(quad, 16, 16, both) == na + nb == 64   # no gap along the diagonal


def test_spec_zero_area_triangle_skipped():                # KN:11-12, 36-37
    tri = np.array([[[1.0, 1.0], [5.0, 5.0], [3.0, 3.0]]])
    out = np.zeros((8, 8), np.uint8)
    assert kn.coverage_fill(tri, 8, 8, out) == 0 and not out.any()


def test_spec_full_viewport_triangle_depth_half():
    tri = np.array([[[-100.0, -100.0], [300.0, -100.0], [-100.0, 300.0]]])
    depth = np.ones((32, 48), np.float32)
    kn.raster_depth(tri, np.zeros((1, 3)), depth)
    assert np.unique(depth).tolist() == [0.5]


def test_empty_inputs():                                   # KN: loops simply do not execute
    out = np.zeros((4, 4), np.uint8)
    assert kn.coverage_fill(np.zeros((0, 3, 2)), 4, 4, out) == 0
    depth = np.ones((4, 4), np.float32)
    assert kn.raster_depth(np.zeros((0, 3, 2)), np.zeros((0, 3)), depth) == 0
    assert (depth == 1.0).all()


# ------------------------------------------------------------------ exact brute force (oracle/brute.py)

@pytest.mark.parametrize("seed", range(6))
def test_oracle_coverage_matches_exact_rational_bruteforce(seed):
    """Second opinion on the C restatement: for triangles on a 1/8-texel grid every product in
    KN:35, 72-74 is exact in float64, so the rational-arithmetic definition (centre inside, top-left
    ties) must give the same coverage plane, owner map and outline -- watertightness included
    (triangles sharing an edge never both cover, and never both miss, a texel on it)."""
    from oracle import brute
    rng = np.random.default_rng(700 + seed)
    w, h, T = 19, 15, 14
    tri = np.round(rng.uniform(-2, 21, size=(T, 3, 2)) * 8.0) / 8.0
    tri[0] = [[2, 2], [12, 2], [2, 12]]                       # two triangles sharing the edge (12,2)-(2,12),
    tri[1] = [[12, 2], [12, 12], [2, 12]]                     # whose centres-on-the-edge test the tie rule
    tri[2, 2] = tri[2, 1]                                     # one degenerate triangle
    ref = np.zeros((h, w), np.uint8)
    n = kn.coverage_fill(tri, w, h, ref)
    want = brute.coverage(tri, w, h)
    assert np.array_equal(ref, want) and n == int(want.sum())
    pair = np.zeros((h, w), np.uint8)
    a = kn.coverage_fill(tri[:1], w, h, pair)
    b = kn.coverage_fill(tri[1:2], w, h, pair)
    assert a + b == int(brute.coverage(tri[:2], w, h).sum())  # no texel of the shared edge counted twice or dropped
    P = rng.normal(size=(T, 3, 3))
    sm = kn.surface_map(tri, P, P, w, h)
    assert np.array_equal(sm["tri_id"], brute.owner(tri, w, h))
    for r in (1, 2):
        assert np.array_equal(kn.outline(want, r), brute.outline(want, r))


# ---- octree baseline kernels: KN:303 expand_pairs_ordered, KN:361 raycast ----

def _icosphere_arrays(level):
    from paper_2501_14807_b200 import synth
    mesh = synth.icosphere_mesh(int(level))
    return (np.ascontiguousarray(mesh.vertices, np.float64),
            np.ascontiguousarray(mesh.triangles, np.int64))


@pytest.mark.parametrize("name", helpers.golden_names("octree_expand"))
def test_oracle_expand_pairs_matches_reference(name):
    f = helpers.golden(name)
    cells, tri = kn.expand_pairs_ordered(f["verts"], f["tris"], f["parent_cells"], f["pair_parent"],
                                         f["pair_tri"], f["cube_min"], float(f["child_h"]))
    assert cells.dtype == np.uint32 and tri.dtype == np.int32
    assert np.array_equal(cells, f["cells"]) and np.array_equal(tri, f["tri"])


@pytest.mark.parametrize("name", helpers.golden_names("octree_scene"))
def test_oracle_octree_build_and_raycast_match_reference(name):
    f = helpers.golden(name)
    verts, tris = _icosphere_arrays(f["level"])
    g = helpers.build_leaf_grid(kn.expand_pairs_ordered, verts, tris, f["cube_min"], float(f["side"]),
                                int(f["depth"]), 2)
    for i, (c, t) in enumerate(g["levels"]):
        assert np.array_equal(c, f["level%d_cells" % (i + 1)])
        assert np.array_equal(t, f["level%d_tri" % (i + 1)])
    assert np.array_equal(g["keys"], f["keys"]) and np.array_equal(g["offsets"], f["offsets"])
    for coarse in (f["coarse"], None):
        for threads in (1, 3):
            bt, btri, leaf = kn.raycast(f["origins"], f["dirs"], f["keys"], f["offsets"], f["tri_idx"],
                                        verts, tris, f["cube_min"], float(f["h"]), int(f["n_cells"]),
                                        coarse, int(f["coarse_shift"]), threads=threads)
            assert np.array_equal(bt, f["best_t"])               # bit-exact incl. inf for misses
            assert np.array_equal(btri, f["best_tri"]) and np.array_equal(leaf, f["leaf_pos"])
    assert np.isfinite(f["best_t"]).sum() > 100 and (f["best_tri"] < 0).sum() > 100


def test_octree_spec_known_answers():
    """depth 0 = one leaf with every triangle; unit cube at depth 1 = all 8 children;
    flat square at z = -0.5 in [-1,1]^3 = exactly the four lower octants."""
    from paper_2501_14807_b200 import synth
    sq = synth.flat_square_mesh(1.0)
    v = np.ascontiguousarray(sq.vertices, np.float64)
    v = (v - v.mean(0)) * 1.6
    v[:, 2] = -0.5
    t = np.ascontiguousarray(sq.triangles, np.int64)
    cells, tri = kn.expand_pairs_ordered(v, t, np.zeros((1, 3), np.uint32), np.zeros(len(t), np.int64),
                                         np.arange(len(t), dtype=np.int32), np.array([-1.0, -1.0, -1.0]), 1.0)
    assert set(map(tuple, cells.tolist())) == {(0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 0)}
    # a face lying exactly on the shared plane z = 0 touches both halves (closed cubes)
    v[:, 2] = 0.0
    cells, _ = kn.expand_pairs_ordered(v, t, np.zeros((1, 3), np.uint32), np.zeros(len(t), np.int64),
                                       np.arange(len(t), dtype=np.int32), np.array([-1.0, -1.0, -1.0]), 1.0)
    assert len(set(map(tuple, cells.tolist()))) == 8
    # empty input (KN:307-309)
    cells, tri = kn.expand_pairs_ordered(v, t, np.zeros((1, 3), np.uint32), np.zeros(0, np.int64),
                                         np.zeros(0, np.int32), np.array([-1.0, -1.0, -1.0]), 1.0)
    assert cells.shape == (0, 3) and tri.shape == (0,)


def test_oracle_raycast_equals_bruteforce_over_all_triangles():
    """Independent of the reference: the DDA traversal must return the globally nearest hit (smallest
    triangle index on ties) -- the same (t, triangle) a brute-force Moeller-Trumbore over every triangle
    finds -- for every ray whose hit lies inside the root cube."""
    from paper_2501_14807_b200 import synth
    rng = np.random.default_rng(77)
    verts, tris = _icosphere_arrays(2)
    verts = verts * np.array([1.0, 0.8, 1.2])
    cube_min, side = helpers.bounding_cube(verts)
    cam = synth.default_camera(40, 40, eye=(0.3, -0.2, 3.0))
    ys, xs = np.mgrid[0:40, 0:40]
    o, d = helpers.camera_rays(cam, np.stack([xs.ravel(), ys.ravel()], 1))
    ro = rng.uniform(-0.4, 0.4, size=(400, 3))                            # origins inside the mesh too
    rd = rng.normal(size=(400, 3))
    origins, dirs = np.concatenate([o, ro]), np.concatenate([d, rd])
    bt, btri = helpers.brute_raycast(origins, dirs, verts, tris)
    for depth in (3, 5):
        g = helpers.build_leaf_grid(kn.expand_pairs_ordered, verts, tris, cube_min, side, depth, 2)
        t, tri, leaf = kn.raycast(origins, dirs, g["keys"], g["offsets"], g["tri_idx"], verts, tris, cube_min,
                                  g["h"], g["n_cells"], g["coarse"], g["coarse_shift"])
        assert np.array_equal(t, bt) and np.array_equal(tri, btri.astype(np.int32))
        assert np.array_equal(leaf >= 0, np.isfinite(bt)) and np.isfinite(bt).sum() > 800


def _sha(a):
    import hashlib
    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), np.uint8)


def test_oracle_matches_reference_on_config_c1_full_size():
    """BASELINE config C1 (icosphere level 5 = 20,480 triangles, 1024^2 atlas, 512^2 window, r = 40 px stroke)
    through all three reference kernels: SHA-256 of every plane and the counts recorded from the reference."""
    f = helpers.golden("c1_digests")
    A, W = int(f["atlas"]), int(f["window"])
    s = helpers.tea_scene_inputs(int(f["level"]), A, W, int(f["tool_r"]), tuple(f["tool_xy"]))
    cov = np.zeros((A, A), np.uint8)
    assert kn.coverage_fill(s["tri_xy"], A, A, cov, threads=0) == int(f["written"])
    assert np.array_equal(_sha(cov), f["cov_sha"])
    depth = np.ones((W, W), np.float32)
    kn.raster_depth(s["win_xy"], s["win_zn"], depth, threads=0)
    assert np.array_equal(_sha(depth), f["depth_sha"])
    data, mask, edited = np.zeros((A, A), np.uint8), np.zeros((A, A), bool), np.zeros((A, A), bool)
    got = kn.raster_tea(s["tri_xy"], s["tri_clip"], float(W), float(W), depth, float(f["eps"]), s["sfx"], s["sfy"],
                        s["bx"], s["by"], s["shape"], data, mask, edited, int(f["value"]), threads=0)
    assert tuple(got) == (int(f["edited_count"]), int(f["fragments"]))
    assert np.array_equal(_sha(data), f["data_sha"]) and np.array_equal(_sha(mask.view(np.uint8)), f["mask_sha"])
    assert np.array_equal(_sha(edited.view(np.uint8)), f["edited_sha"])


def test_oracle_matches_reference_on_config_c2_mesh():
    """BASELINE config C2's mesh (999,698 triangles, 4096^2 atlas, 1024^2 window, r = 70 px stroke): the
    reference needed ~10 minutes of numpy loops for these digests (make_golden.py --c2)."""
    if "c2_digests" not in helpers.golden_names("c2_"):
        pytest.skip("tests/golden/c2_digests.npz not generated (python tests/golden/make_golden.py --c2)")
    f = helpers.golden("c2_digests")
    A, W = int(f["atlas"]), int(f["window"])
    s = helpers.terrain_scene_inputs(int(f["quads"]), A, W, int(f["tool_r"]))
    assert s["mesh"].num_triangles == int(f["triangles"])
    cov = np.zeros((A, A), np.uint8)
    assert kn.coverage_fill(s["tri_xy"], A, A, cov, threads=0) == int(f["written"])
    assert np.array_equal(_sha(cov), f["cov_sha"])
    depth = np.ones((W, W), np.float32)
    kn.raster_depth(s["win_xy"], s["win_zn"], depth, threads=0)
    assert np.array_equal(_sha(depth), f["depth_sha"])
    data, mask, edited = np.zeros((A, A), np.uint8), np.zeros((A, A), bool), np.zeros((A, A), bool)
    got = kn.raster_tea(s["tri_xy"], s["tri_clip"], float(W), float(W), depth, float(f["eps"]), s["sfx"], s["sfy"],
                        s["bx"], s["by"], s["shape"], data, mask, edited, int(f["value"]), threads=0)
    assert tuple(got) == (int(f["edited_count"]), int(f["fragments"]))
    assert np.array_equal(_sha(data), f["data_sha"]) and np.array_equal(_sha(mask.view(np.uint8)), f["mask_sha"])
    assert np.array_equal(_sha(edited.view(np.uint8)), f["edited_sha"])


def _octree_digest_scene(f):
    verts, tris = _icosphere_arrays(f["level"])
    cube_min, side = helpers.bounding_cube(verts)
    origins, dirs = helpers.octree_rays(int(f["window"]), int(f["seed"]), int(f["nrandom"]))
    return verts, tris, cube_min, side, origins, dirs


def test_oracle_matches_reference_on_larger_octree_scene():
    """20,480 triangles, depth 8 (307,904 leaves, 549,464 rows), 20,480 rays: digests of the reference's leaf
    arrays and ray-cast results (make_golden.py --octree)."""
    f = helpers.golden("octree_digests")
    verts, tris, cube_min, side, origins, dirs = _octree_digest_scene(f)
    g = helpers.build_leaf_grid(kn.expand_pairs_ordered, verts, tris, cube_min, side, int(f["depth"]), int(f["coarse_bits"]))
    assert [len(t) for _, t in g["levels"]] == f["level_rows"].tolist()
    assert np.array_equal(_sha(g["keys"]), f["keys_sha"]) and np.array_equal(_sha(g["offsets"]), f["offsets_sha"])
    assert np.array_equal(_sha(g["tri_idx"]), f["tri_idx_sha"])
    bt, btri, leaf = kn.raycast(origins, dirs, g["keys"], g["offsets"], g["tri_idx"], verts, tris, cube_min, g["h"],
                                g["n_cells"], g["coarse"], g["coarse_shift"], threads=0)
    assert int(np.isfinite(bt).sum()) == int(f["hits"])
    assert np.array_equal(_sha(bt), f["best_t_sha"]) and np.array_equal(_sha(btri), f["best_tri_sha"])
    assert np.array_equal(_sha(leaf), f["leaf_sha"])


def test_oracle_matches_reference_on_c1_stroke_session():
    """Eight strokes accumulating in one layer on config C1 (make_golden.py --session): counts of every stroke
    and plane digests after every stroke equal the reference's."""
    f = helpers.golden("c1_session_digests")
    A, W = int(f["atlas"]), int(f["window"])
    s = helpers.tea_scene_inputs(5, A, W, 10, (W / 2.0, W / 2.0))
    depth = np.ones((W, W), np.float32)
    kn.raster_depth(s["win_xy"], s["win_zn"], depth, threads=0)
    data, mask = np.zeros((A, A), np.uint8), np.zeros((A, A), bool)
    for k, st in enumerate(helpers.c1_stroke_script(W)):
        shape, (sfx, sfy, bx, by) = helpers.stroke_tool_map(st, W)
        edited = np.zeros((A, A), bool)
        got = kn.raster_tea(s["tri_xy"], s["tri_clip"], float(W), float(W), depth, 1e-4, sfx, sfy, bx, by, shape,
                            data, mask, edited, st["value"], threads=0)
        assert tuple(got) == tuple(f["counts"][k])
        assert np.array_equal(_sha(data), f["data_sha"][k]) and np.array_equal(_sha(mask.view(np.uint8)), f["mask_sha"][k])
        assert np.array_equal(_sha(edited.view(np.uint8)), f["edited_sha"][k])
