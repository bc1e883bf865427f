"""GPU parity of the three reference kernels (coverage_fill / raster_depth / raster_tea) called
through the C ABI: against the reference's own outputs (golden fixtures) and against the oracle
on random scenes.  Bit-exact for every plane; counts exact where the reference's are order-free."""
import numpy as np
import pytest

import helpers
from oracle import kn
from paper_2501_14807_b200 import _native as nat

pytestmark = pytest.mark.gpu


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _plane_dev(a):
    import torch
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        return torch.from_numpy(a.view(np.int32)).cuda().view(torch.uint32)
    return torch.from_numpy(a).cuda()


def _host(t):
    import torch
    if t.dtype == torch.uint32:
        return t.view(torch.int32).cpu().numpy().view(np.uint32)
    return t.cpu().numpy()


# ------------------------------------------------------------------ golden fixtures

@pytest.mark.parametrize("name", helpers.golden_names("coverage_"))
@pytest.mark.parametrize("path", ["host", "device"])
def test_coverage_golden(name, path):
    g = helpers.golden(name)
    w, h = int(g["width"]), int(g["height"])
    if path == "host":
        out = g["out0"].copy()
        written = nat.coverage_fill(g["tri_xy"], w, h, out)
    else:
        d = _dev(g["out0"])
        written = nat.coverage_fill(_dev(g["tri_xy"]), w, h, d)
        out = d.cpu().numpy()
    assert np.array_equal(out, g["out"])
    assert written == int(g["written"])


@pytest.mark.parametrize("name", helpers.golden_names("depth_"))
@pytest.mark.parametrize("path", ["host", "device"])
def test_depth_golden(name, path):
    g = helpers.golden(name)
    if path == "host":
        depth = g["depth0"].copy()
        nat.raster_depth(g["tri_xy"], g["tri_zn"], depth)
    else:
        d = _dev(g["depth0"])
        nat.raster_depth(_dev(g["tri_xy"]), _dev(g["tri_zn"]), d)
        depth = d.cpu().numpy()
    assert np.array_equal(depth.view(np.uint32), g["depth"].view(np.uint32))


@pytest.mark.parametrize("name", helpers.golden_names("tea_rand_"))
@pytest.mark.parametrize("path", ["host", "device"])
def test_tea_random_golden(name, path):
    g = helpers.golden(name)
    args = (float(g["ww"]), float(g["wh"]), g["depth"], helpers.eps_of(g), float(g["sfx"]), float(g["sfy"]),
            float(g["bx"]), float(g["by"]), g["shape"])
    if path == "host":
        data, mask, edited = g["data0"].copy(), g["mask0"].copy(), g["edited0"].copy()
        ec, fr = nat.raster_tea(g["tri_xy"], g["tri_clip"], *args, data, mask, edited, g["value"][()])
    else:
        d, m, e = _plane_dev(g["data0"]), _dev(g["mask0"]), _dev(g["edited0"])
        ec, fr = nat.raster_tea(_dev(g["tri_xy"]), _dev(g["tri_clip"]), *args, d, m, e, g["value"][()])
        data, mask, edited = _host(d), m.cpu().numpy(), e.cpu().numpy()
    assert (ec, fr) == (int(g["edited_count"]), int(g["fragments"]))
    assert np.array_equal(data.view(np.uint8), g["data"].view(np.uint8))
    assert np.array_equal(mask, g["mask"])
    assert np.array_equal(edited, g["edited"])


@pytest.mark.parametrize("name", helpers.golden_names("tea_scene_"))
def test_tea_scene_golden_direct_and_cached(name):
    """Reference outputs reproduced by BOTH TEA kernels (direct per-triangle, and per-texel over
    the cached triangle-id map) on a real camera / mesh / atlas scene."""
    import torch
    g = helpers.golden(name)
    s = helpers.tea_scene_inputs(g["level"], g["atlas"], g["window"], g["tool_r"], g["tool_xy"])
    A, W = int(g["atlas"]), int(g["window"])
    depth = torch.ones((W, W), dtype=torch.float32, device="cuda")
    nat.raster_depth(_dev(s["win_xy"]), _dev(s["win_zn"]), depth)
    assert np.array_equal(depth.cpu().numpy().view(np.uint32), g["depth"].view(np.uint32))
    tri_xy, tri_clip = _dev(s["tri_xy"]), _dev(s["tri_clip"])
    tri_id, frags, overlap = nat.raster_tri_id(tri_xy, A, A)
    assert overlap == 0 and frags == int(g["cov_count"])
    for cached in (False, True):
        data = torch.zeros((A, A), dtype=torch.uint8, device="cuda")
        mask = torch.zeros((A, A), dtype=torch.bool, device="cuda")
        edited = torch.zeros((A, A), dtype=torch.bool, device="cuda")
        args = (float(W), float(W), depth, helpers.eps_of(g), s["sfx"], s["sfy"], s["bx"], s["by"], s["shape"],
                data, mask, edited, 7)
        ec, fr = nat.tea_texels(tri_xy, tri_clip, tri_id, *args) if cached else nat.raster_tea(tri_xy, tri_clip, *args)
        assert (ec, fr) == (int(g["edited_count"]), int(g["fragments"]))
        assert np.array_equal(np.packbits(mask.cpu().numpy()), g["mask"])
        assert np.array_equal(np.packbits(edited.cpu().numpy()), g["edited"])
        d = data.cpu().numpy()
        assert np.array_equal(np.packbits(d != 0), g["data"]) and set(np.unique(d)) <= {0, 7}


def test_eps_promotion_mode_golden():
    g = helpers.golden("epsmode")
    got = []
    for e in (float(g["eps"]), np.float64(g["eps"])):
        data, mask, edited = np.zeros((4, 4), np.uint8), np.zeros((4, 4), bool), np.zeros((4, 4), bool)
        depth = np.full((4, 4), g["depth_value"], np.float32)
        got.append(nat.raster_tea(g["tri_xy"], g["tri_clip"], 4.0, 4.0, depth, e, 0.5, 0.5, 0.5, 0.5,
                                  np.ones((1, 1), np.uint8), data, mask, edited, 1)[0])
    assert got == [int(g["edited_weak"]), int(g["edited_f64"])]


# ------------------------------------------------------------------ random scenes vs the oracle

@pytest.mark.parametrize("seed", range(6))
def test_coverage_span_path_dirty_misaligned(seed):
    """Row-span rasteriser (few, large triangles -> the span variant) writing byte planes word by
    word: odd widths, a plane view starting at an odd byte offset, planes pre-dirtied with values
    other than 0 / 1 (KN:97-99 sets them to exactly 1 and does not count them), overlapping
    triangles racing on the same words; the texel-walk variant (many small triangles) agrees."""
    import torch
    from paper_2501_14807_b200 import synth
    rng = np.random.default_rng(3000 + seed)
    w, h = int(rng.integers(61, 260)) | 1, int(rng.integers(40, 200))
    ntri = 40
    tri = synth.random_soup(rng, ntri, float(max(w, h)), dtype=np.float64, degenerate_frac=0.05, snap_frac=0.5)
    dirty = rng.choice(np.array([0, 0, 0, 1, 2, 255], np.uint8), size=(h, w))
    ref = dirty.copy()
    want = kn.coverage_fill(tri, w, h, ref)
    off = int(rng.integers(1, 4))
    buf = torch.zeros(h * w + 8, dtype=torch.uint8, device="cuda")
    out = buf[off:off + h * w].view(h, w)
    out.copy_(_dev(dirty))
    assert nat.coverage_fill(_dev(tri), w, h, out) == want
    assert np.array_equal(out.cpu().numpy(), ref)
    assert not bool(buf[:off].any()) and not bool(buf[off + h * w:].any())          # neighbours of the view untouched
    # same scene cut into many small triangles takes the texel-walk variant: same plane
    small = synth.random_soup(rng, 4000, float(max(w, h)), dtype=np.float64)
    ref2 = dirty.copy()
    want2 = kn.coverage_fill(small, w, h, ref2)
    out.copy_(_dev(dirty))
    assert nat.coverage_fill(_dev(small), w, h, out) == want2 and np.array_equal(out.cpu().numpy(), ref2)


@pytest.mark.parametrize("seed", range(8))
def test_coverage_random_vs_oracle(seed):
    from paper_2501_14807_b200 import synth
    rng = np.random.default_rng(1000 + seed)
    w, h = int(rng.integers(20, 200)), int(rng.integers(20, 200))
    tri = synth.random_soup(rng, 400, float(max(w, h)), dtype=np.float32 if seed % 2 else np.float64)
    ref = np.zeros((h, w), np.uint8)
    want = kn.coverage_fill(tri, w, h, ref)
    out = _dev(np.zeros((h, w), np.uint8))
    got = nat.coverage_fill(_dev(tri), w, h, out)
    assert got == want and np.array_equal(out.cpu().numpy(), ref)
    # permutation invariance on the GPU path
    out2 = _dev(np.zeros((h, w), np.uint8))
    assert nat.coverage_fill(_dev(tri[rng.permutation(len(tri))]), w, h, out2) == want
    assert np.array_equal(out2.cpu().numpy(), ref)


@pytest.mark.parametrize("seed", range(6))
def test_depth_random_vs_oracle(seed):
    from paper_2501_14807_b200 import synth
    rng = np.random.default_rng(2000 + seed)
    w, h = int(rng.integers(20, 150)), int(rng.integers(20, 150))
    tri = synth.random_soup(rng, 500, float(max(w, h)))
    zn = rng.uniform(-1.5, 1.2, size=(500, 3))
    ref = np.ones((h, w), np.float32)
    kn.raster_depth(tri, zn, ref)
    d = _dev(np.ones((h, w), np.float32))
    changed = nat.raster_depth(_dev(tri), _dev(zn), d)
    assert np.array_equal(d.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    assert changed == int((ref != 1.0).sum())


@pytest.mark.parametrize("seed", range(20))
def test_tea_random_vs_oracle(seed):
    """SPEC.md:605 acceptance #1 scale: >= 20 random scenes, all plane kinds."""
    kinds = [(np.uint8, 200), (np.int8, -7), (np.int16, 3000), (np.int32, -123456), (np.uint32, 3123456789),
             (np.float16, 1.5), (np.float32, -0.25)]
    dt, val = kinds[seed % len(kinds)]
    c = helpers.random_tea_case(3000 + seed, ntri=300 + 30 * seed, w=96, h=128, plane_dtype=dt, value=val,
                                tri_dtype=np.float32 if seed % 3 == 0 else np.float64,
                                eps=np.float64(1e-4) if seed % 4 == 1 else 1e-4)
    rd, rm, re = c["data"].copy(), c["mask"].copy(), c["edited"].copy()
    want = kn.raster_tea(*helpers.tea_args(c), rd, rm, re, val)
    d, m, e = _plane_dev(c["data"]), _dev(c["mask"]), _dev(c["edited"])
    got = nat.raster_tea(_dev(c["tri_xy"]), _dev(c["tri_clip"]), *helpers.tea_args(c)[2:], d, m, e, val)
    assert got == want
    assert np.array_equal(_host(d).view(np.uint8), rd.view(np.uint8))
    assert np.array_equal(m.cpu().numpy(), rm) and np.array_equal(e.cpu().numpy(), re)


@pytest.mark.parametrize("seed", range(14))
def test_host_plane_twins_vs_oracle(seed):
    """The host-buffer twins (numpy planes, KN call shape): nothing of the caller's planes is uploaded, the
    written SET comes back as a bitmap (dense strokes) or as a word list (sparse strokes) and is applied to
    pre-dirtied host planes.  Ragged plane sizes (texel count not a multiple of 64), float32 and float64
    triangles, every plane kind, planes holding bytes other than 0 / 1."""
    kinds = [(np.uint8, 200), (np.int8, -7), (np.int16, 3000), (np.int32, -123456), (np.uint32, 3123456789),
             (np.float16, 1.5), (np.float32, -0.25)]
    dt, val = kinds[seed % len(kinds)]
    w, h = [(96, 128), (50, 37), (129, 65), (64, 64)][seed % 4]
    c = helpers.random_tea_case(5000 + seed, ntri=40 if seed % 2 else 900, w=w, h=h, plane_dtype=dt, value=val,
                                tri_dtype=np.float32 if seed % 3 == 0 else np.float64)
    rng = np.random.default_rng(seed)
    dirty = rng.integers(0, 4, size=(h, w)).astype(np.uint8) * (rng.random((h, w)) < 0.2)      # bytes 0..3
    c["edited"] = dirty.copy()
    rd, rm, re = c["data"].copy(), c["mask"].copy(), c["edited"].copy()
    want = kn.raster_tea(*helpers.tea_args(c), rd, rm, re, val)
    d, m, e = c["data"].copy(), c["mask"].copy(), c["edited"].copy()
    got = nat.raster_tea(*helpers.tea_args(c), d, m, e, val)
    assert got == want
    assert np.array_equal(d.view(np.uint8), rd.view(np.uint8)) and np.array_equal(m, rm) and np.array_equal(e, re)
    # coverage_fill into a dirty plane, and twice (second call writes nothing new)
    out, ref = dirty.copy(), dirty.copy()
    assert nat.coverage_fill(c["tri_xy"], w, h, out) == kn.coverage_fill(c["tri_xy"], w, h, ref)
    assert np.array_equal(out, ref)
    assert nat.coverage_fill(c["tri_xy"], w, h, out) == 0 and np.array_equal(out, ref)


def test_tea_idempotent():
    c = helpers.random_tea_case(77, ntri=200, w=64, h=64)
    d, m, e = _plane_dev(c["data"]), _dev(c["mask"]), _dev(np.zeros((64, 64), np.uint8))
    a = (_dev(c["tri_xy"]), _dev(c["tri_clip"])) + helpers.tea_args(c)[2:]
    first = nat.raster_tea(*a, d, m, e, 9)
    snap = (d.clone(), m.clone(), e.clone())
    second = nat.raster_tea(*a, d, m, e, 9)
    assert second == (0, first[1])
    assert all(bool((x == y).all()) for x, y in zip(snap, (d, m, e)))


def test_large_and_small_triangles_mix():
    """Exercises all three raster passes: warp-per-triangle, the scan, and block chunks for
    triangles far larger than SMALL_MAX texels (incl. two that tile the whole plane)."""
    rng = np.random.default_rng(5)
    w = h = 700
    big = np.array([[[0, 0], [w, 0], [w, h]], [[0, 0], [w, h], [0, h]]], dtype=np.float64)
    mid = rng.uniform(0, w, size=(40, 3, 2))
    small = rng.uniform(0, w, size=(3000, 1, 2)) + rng.normal(size=(3000, 3, 2)) * 2.0
    tri = np.concatenate([small[:1500], mid, big, small[1500:]])
    ref = np.zeros((h, w), np.uint8)
    want = kn.coverage_fill(tri, w, h, ref, threads=4)
    out = _dev(np.zeros((h, w), np.uint8))
    assert nat.coverage_fill(_dev(tri), w, h, out) == want == w * h
    assert np.array_equal(out.cpu().numpy(), ref)
    zn = rng.uniform(-1, 1, size=(len(tri), 3))
    dref = np.ones((h, w), np.float32)
    kn.raster_depth(tri, zn, dref, threads=4)
    d = _dev(np.ones((h, w), np.float32))
    nat.raster_depth(_dev(tri), _dev(zn), d)
    assert np.array_equal(d.cpu().numpy().view(np.uint32), dref.view(np.uint32))


def test_row_slabs_concatenate_to_full_plane():
    """Row sharding (SURVEY.md 4 'distributed testing without a cluster'): logical slabs on one
    GPU concatenate to the unsharded result bit-for-bit; counts add up."""
    c = helpers.random_tea_case(91, ntri=400, w=80, h=120)
    rd, rm, re = c["data"].copy(), c["mask"].copy(), c["edited"].copy()
    want = kn.raster_tea(*helpers.tea_args(c), rd, rm, re, 5)
    tri, clip = _dev(c["tri_xy"]), _dev(c["tri_clip"])
    ec = fr = 0
    parts = []
    for r0, r1 in ((0, 37), (37, 38), (38, 120)):
        d, m, e = _plane_dev(c["data"][r0:r1]), _dev(c["mask"][r0:r1]), _dev(c["edited"][r0:r1])
        a, b = nat.raster_tea(tri, clip, *helpers.tea_args(c)[2:], d, m, e, 5, height=120, row0=r0)
        ec, fr = ec + a, fr + b
        parts.append((d.cpu().numpy(), m.cpu().numpy(), e.cpu().numpy()))
    assert (ec, fr) == want
    for k, ref in enumerate((rd, rm, re)):
        assert np.array_equal(np.concatenate([p[k] for p in parts]), ref)


def test_empty_and_degenerate_inputs():
    import torch
    out = torch.zeros((8, 8), dtype=torch.uint8, device="cuda")
    assert nat.coverage_fill(_dev(np.zeros((0, 3, 2))), 8, 8, out) == 0
    deg = np.array([[[1.0, 1.0], [5.0, 5.0], [3.0, 3.0]], [[np.nan, 0, ], [1, 1], [2, 0]]])
    assert nat.coverage_fill(_dev(deg), 8, 8, out) == 0 and not bool(out.any())
    assert nat.coverage_fill(np.zeros((0, 3, 2)), 8, 8, np.zeros((8, 8), np.uint8)) == 0


@pytest.mark.parametrize("seed", range(4))
def test_cuda_rasteriser_matches_exact_rational_bruteforce(seed):
    """The CUDA rasteriser (span and texel-walk variants) against the exact rational-arithmetic brute
    force of oracle/brute.py on 1/8-texel-grid triangles: coverage plane, count and owner map."""
    from oracle import brute
    rng = np.random.default_rng(800 + seed)
    w, h = 40, 33
    T = 6 if seed % 2 else 60                                  # few large (span variant) / many small triangles
    scale = 30.0 if seed % 2 else 9.0
    c = rng.uniform(0, 40, size=(T, 1, 2))
    tri = np.round((c + rng.normal(size=(T, 3, 2)) * scale) * 8.0) / 8.0
    want = brute.coverage(tri, w, h)
    out = _dev(np.zeros((h, w), np.uint8))
    assert nat.coverage_fill(_dev(tri), w, h, out) == int(want.sum())
    assert np.array_equal(out.cpu().numpy(), want)
    tri_id, frags, overlap = nat.raster_tri_id(_dev(tri), w, h)
    assert np.array_equal(tri_id.cpu().numpy(), brute.owner(tri, w, h))
    assert frags - overlap == int(want.sum())


def test_cuda_matches_reference_on_config_c1_full_size():
    """BASELINE config C1 at full size against the REFERENCE's recorded plane digests (tests/golden/
    c1_digests.npz): host-buffer twins of all three kernels, and the resident stroke pipeline."""
    import hashlib
    import paper_2501_14807_b200 as ml
    from paper_2501_14807_b200 import synth

    def sha(a):
        return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), np.uint8)
    f = helpers.golden("c1_digests")
    A, W = int(f["atlas"]), int(f["window"])
    s = helpers.tea_scene_inputs(int(f["level"]), A, W, int(f["tool_r"]), tuple(f["tool_xy"]))
    cov = np.zeros((A, A), np.uint8)
    assert nat.coverage_fill(s["tri_xy"], A, A, cov) == int(f["written"]) and np.array_equal(sha(cov), f["cov_sha"])
    depth = np.ones((W, W), np.float32)
    nat.raster_depth(s["win_xy"], s["win_zn"], depth)
    assert np.array_equal(sha(depth), f["depth_sha"])
    data, mask, edited = np.zeros((A, A), np.uint8), np.zeros((A, A), bool), np.zeros((A, A), bool)
    got = nat.raster_tea(s["tri_xy"], s["tri_clip"], float(W), float(W), depth, float(f["eps"]), s["sfx"], s["sfy"],
                       s["bx"], s["by"], s["shape"], data, mask, edited, int(f["value"]))
    assert tuple(got) == (int(f["edited_count"]), int(f["fragments"]))
    assert np.array_equal(sha(data), f["data_sha"]) and np.array_equal(sha(mask.view(np.uint8)), f["mask_sha"])
    assert np.array_equal(sha(edited.view(np.uint8)), f["edited_sha"])
    # the resident pipeline (surface map + render_depth + culled apply_stroke) lands on the same planes
    mesh, cam = s["mesh"], s["cam"]
    surf = ml.build_surface_map(mesh, A, A)
    dmap = ml.render_depth(mesh, cam)
    assert np.array_equal(sha(dmap.plane.cpu().numpy()), f["depth_sha"])
    assert np.array_equal(sha(surf.coverage.cpu().numpy().astype(np.uint8)), f["cov_sha"])
    ctx = ml.StrokeContext(mesh, cam, dmap, surf)
    layer = ml.create_layer("c1", "uint8", A, A, pool=ml.TexturePool())
    tool = ml.EditingTool(px=float(f["tool_xy"][0]), py=float(f["tool_xy"][1]), shape=synth.circle_shape(int(f["tool_r"])),
                          value=int(f["value"]))
    res = ml.apply_stroke(ctx, tool, layer)
    assert (res.edited_count, res.fragments) == (int(f["edited_count"]), int(f["fragments"]))
    assert np.array_equal(sha(layer.data.cpu().numpy()), f["data_sha"])
    assert np.array_equal(sha(layer.mask.cpu().numpy().view(np.uint8)), f["mask_sha"])
    assert np.array_equal(sha(res.edited_mask.cpu().numpy().view(np.uint8)), f["edited_sha"])


def test_cuda_matches_reference_on_config_c2_mesh():
    """BASELINE config C2's mesh (999,698 triangles, 4096^2 atlas, 1024^2 window, r = 70 px) against the
    REFERENCE's recorded plane digests (tests/golden/c2_digests.npz, ~10 min of reference time): host-buffer
    twins of all three kernels, and the resident stroke pipeline."""
    import hashlib
    import paper_2501_14807_b200 as ml
    from paper_2501_14807_b200 import synth

    def sha(a):
        return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), np.uint8)
    if "c2_digests" not in helpers.golden_names("c2_"):
        pytest.skip("tests/golden/c2_digests.npz not generated (python tests/golden/make_golden.py --c2)")
    f = helpers.golden("c2_digests")
    A, W = int(f["atlas"]), int(f["window"])
    s = helpers.terrain_scene_inputs(int(f["quads"]), A, W, int(f["tool_r"]))
    cov = np.zeros((A, A), np.uint8)
    assert nat.coverage_fill(s["tri_xy"], A, A, cov) == int(f["written"]) and np.array_equal(sha(cov), f["cov_sha"])
    depth = np.ones((W, W), np.float32)
    nat.raster_depth(s["win_xy"], s["win_zn"], depth)
    assert np.array_equal(sha(depth), f["depth_sha"])
    data, mask, edited = np.zeros((A, A), np.uint8), np.zeros((A, A), bool), np.zeros((A, A), bool)
    got = nat.raster_tea(s["tri_xy"], s["tri_clip"], float(W), float(W), depth, float(f["eps"]), s["sfx"], s["sfy"],
                       s["bx"], s["by"], s["shape"], data, mask, edited, int(f["value"]))
    assert tuple(got) == (int(f["edited_count"]), int(f["fragments"]))
    assert np.array_equal(sha(data), f["data_sha"]) and np.array_equal(sha(mask.view(np.uint8)), f["mask_sha"])
    assert np.array_equal(sha(edited.view(np.uint8)), f["edited_sha"])
    # the resident pipeline (surface map + render_depth + culled apply_stroke) lands on the same planes
    mesh, cam = s["mesh"], s["cam"]
    surf = ml.build_surface_map(mesh, A, A)
    dmap = ml.render_depth(mesh, cam)
    assert np.array_equal(sha(dmap.plane.cpu().numpy()), f["depth_sha"])
    assert np.array_equal(sha(surf.coverage.cpu().numpy().astype(np.uint8)), f["cov_sha"])
    ctx = ml.StrokeContext(mesh, cam, dmap, surf)
    layer = ml.create_layer("c2", "uint8", A, A, pool=ml.TexturePool())
    tool = ml.EditingTool(px=0.5 * W, py=0.5 * W, shape=synth.circle_shape(int(f["tool_r"])),
                          value=int(f["value"]))
    res = ml.apply_stroke(ctx, tool, layer)
    assert (res.edited_count, res.fragments) == (int(f["edited_count"]), int(f["fragments"]))
    assert np.array_equal(sha(layer.data.cpu().numpy()), f["data_sha"])
    assert np.array_equal(sha(layer.mask.cpu().numpy().view(np.uint8)), f["mask_sha"])
    assert np.array_equal(sha(res.edited_mask.cpu().numpy().view(np.uint8)), f["edited_sha"])


def test_cuda_stroke_session_matches_reference_digests():
    """Eight strokes accumulating in one layer on config C1 through the resident pipeline -- culled, streamed
    and direct TEA kernels interleaved on ONE context, so the per-stroke reset of the edited mask (SPEC:253-255,
    done tile-wise by the culled path) is exercised -- against the REFERENCE's per-stroke counts and plane
    digests (tests/golden/c1_session_digests.npz)."""
    import hashlib
    import paper_2501_14807_b200 as ml

    def sha(a):
        return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), np.uint8)
    f = helpers.golden("c1_session_digests")
    A, W = int(f["atlas"]), int(f["window"])
    s = helpers.tea_scene_inputs(5, A, W, 10, (W / 2.0, W / 2.0))
    mesh, cam = s["mesh"], s["cam"]
    ctx = ml.StrokeContext(mesh, cam, ml.render_depth(mesh, cam), ml.build_surface_map(mesh, A, A))
    layer = ml.create_layer("session", "uint8", A, A, pool=ml.TexturePool())
    modes = ["cull", "cull", "stream", "cull", "direct", "cull", "cull", "stream"]
    for k, st in enumerate(helpers.c1_stroke_script(W)):
        shape, _ = helpers.stroke_tool_map(st, W)
        tool = ml.EditingTool(px=st["px"], py=st["py"], shape=shape, value=st["value"])
        res = ml.apply_stroke(ctx, tool, layer, cull=(modes[k] == "cull"), force_direct=(modes[k] == "direct"))
        assert (res.edited_count, res.fragments) == tuple(f["counts"][k]), (k, modes[k])
        assert np.array_equal(sha(layer.data.cpu().numpy()), f["data_sha"][k]), (k, modes[k])
        assert np.array_equal(sha(layer.mask.cpu().numpy().view(np.uint8)), f["mask_sha"][k]), (k, modes[k])
        assert np.array_equal(sha(res.edited_mask.cpu().numpy().view(np.uint8)), f["edited_sha"][k]), (k, modes[k])
