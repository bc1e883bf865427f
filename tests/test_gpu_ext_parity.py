"""GPU parity of the north-star operations (surface map, sphere / threshold selection, layer
algebra, areas, outline / padding) against their frozen definitions in oracle/kn_port.c.
Integer / byte planes bit-exact; float32 maps bit-exact (tighter than the 1e-5 the north star
asks); areas within 1e-10 relative (north star: 1e-6)."""
import numpy as np
import pytest

import helpers
from oracle import kn
from paper_2501_14807_b200 import _native as nat
from paper_2501_14807_b200 import synth

pytestmark = pytest.mark.gpu


def _dev(a):
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


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def _mesh_arrays(mesh, w, h):
    return mesh.tri_uv_texels(w, h), mesh.tri_pos(), mesh.tri_nrm()


@pytest.fixture(scope="module")
def sphere_map():
    """Icosphere level 3 (1,280 triangles) in a 256^2 chart-grid atlas: oracle + GPU surface maps."""
    mesh = synth.icosphere_mesh(3)
    w = h = 256
    xy, P, N = _mesh_arrays(mesh, w, h)
    ref = kn.surface_map(xy, P, N, w, h)
    got = nat.surface_map(xy, P, N, w, h)
    return mesh, ref, got


def test_surface_map_bit_exact(sphere_map):
    _, ref, got = sphere_map
    assert got["covered"] == ref["covered"] and got["overlap"] == ref["overlap"] == 0
    assert np.array_equal(got["tri_id"].cpu().numpy(), ref["tri_id"])
    for k in ("pos", "nrm", "area"):
        assert np.array_equal(_bits(got[k].cpu().numpy()), _bits(ref[k])), k
    # uncovered texels: NaN position, zero normal / area
    unc = ref["tri_id"] < 0
    assert np.isnan(got["pos"].cpu().numpy()[:, unc]).all()


def test_surface_map_overlap_soup_and_f32_inputs():
    rng = np.random.default_rng(9)
    w, h = 150, 90
    xy = synth.random_soup(rng, 300, float(w)).astype(np.float32)
    P = rng.normal(size=(300, 3, 3)).astype(np.float32)
    N = rng.normal(size=(300, 3, 3)).astype(np.float32)
    ref = kn.surface_map(xy, P, N, w, h)
    got = nat.surface_map(xy, P, N, w, h)
    assert got["overlap"] == ref["overlap"] > 0 and got["covered"] == ref["covered"]
    assert np.array_equal(got["tri_id"].cpu().numpy(), ref["tri_id"])
    for k in ("pos", "nrm", "area"):
        assert np.array_equal(_bits(got[k].cpu().numpy()), _bits(ref[k])), k


def test_surface_map_area_anchors():
    """a 1 m^2 flat square fully covering a 64^2 atlas -> every texel carries
    1/64^2 m^2, the layer area of a full mask is the mesh area, precision = area / texels."""
    import torch
    from paper_2501_14807_b200 import TriangleMesh, mesh_surface_area
    mesh = TriangleMesh(vertices=np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], float),
                        normals=np.array([[0, 0, 1]] * 4, float),
                        uvs=np.array([[0, 0], [1, 0], [1, 1], [0, 1]], float),
                        triangles=np.array([[0, 1, 2], [0, 2, 3]]))
    assert mesh_surface_area(mesh) == 1.0
    got = nat.surface_map(*_mesh_arrays(mesh, 64, 64), 64, 64)
    assert got["covered"] == 4096
    full = torch.ones((64, 64), dtype=torch.uint8, device="cuda")
    sums, counts = nat.layer_area(got["area"], [full])
    assert counts[0] == 4096 and abs(sums[0] - 1.0) < 1e-9
    assert abs(sums[0] / counts[0] * 1e4 - 1e4 / 64 ** 2) < 1e-9        # cm^2 per texel


def test_surface_map_row_slabs(sphere_map):
    mesh, ref, _ = sphere_map
    xy, P, N = _mesh_arrays(mesh, 256, 256)
    parts = [nat.surface_map(xy, P, N, 256, 256, row0=r0, rows=r1 - r0) for r0, r1 in ((0, 100), (100, 101), (101, 256))]
    assert sum(p["covered"] for p in parts) == ref["covered"]
    assert np.array_equal(np.concatenate([p["tri_id"].cpu().numpy() for p in parts]), ref["tri_id"])
    pos = np.concatenate([p["pos"].cpu().numpy() for p in parts], axis=1)
    assert np.array_equal(_bits(pos), _bits(ref["pos"]))


@pytest.mark.parametrize("kind,value", [(np.uint8, 9), (np.int16, -5), (np.uint32, 77777), (np.float32, 0.5)])
def test_select_sphere_bit_exact(sphere_map, kind, value):
    _, ref, got = sphere_map
    rng = np.random.default_rng(3)
    for center, radius in (((0.0, 0.0, 1.0), 0.25), ((0.6, -0.5, 0.3), 0.6), ((5.0, 5.0, 5.0), 0.1), ((0, 0, 0), 2.0)):
        data0 = rng.integers(0, 4, size=(256, 256)).astype(kind)
        mask0 = rng.random((256, 256)) < 0.2
        ed0 = (rng.random((256, 256)) < 0.1).astype(np.uint8)
        rd, rm, re = data0.copy(), mask0.copy(), ed0.copy()
        want = kn.select_sphere(ref["pos"], center, radius, rd, rm, re, value)
        d, m, e = _dev(data0), _dev(mask0), _dev(ed0)
        assert nat.select_sphere(got["pos"], center, radius, d, m, e, value) == want
        assert np.array_equal(_bits(_host(d)), _bits(rd))
        assert np.array_equal(m.cpu().numpy(), rm) and np.array_equal(e.cpu().numpy(), re)


def test_select_sphere_unaligned_and_tail():
    """n not a multiple of 4 and planes at odd offsets take the scalar path."""
    import torch
    rng = np.random.default_rng(4)
    n_rows, w = 7, 37
    pos = rng.normal(size=(3, n_rows, w)).astype(np.float32)
    pos[:, rng.random((n_rows, w)) < 0.2] = np.nan
    rd = np.zeros((n_rows, w), np.uint8); rm = np.zeros((n_rows, w), bool); re = np.zeros((n_rows, w), np.uint8)
    want = kn.select_sphere(pos, (0.1, 0.2, -0.1), 0.9, rd, rm, re, 3)
    d = torch.zeros((n_rows, w), dtype=torch.uint8, device="cuda")
    m = torch.zeros((n_rows, w), dtype=torch.bool, device="cuda")
    e = torch.zeros((n_rows, w), dtype=torch.uint8, device="cuda")
    assert nat.select_sphere(_dev(pos), (0.1, 0.2, -0.1), 0.9, d, m, e, 3) == want
    assert np.array_equal(d.cpu().numpy(), rd) and np.array_equal(m.cpu().numpy(), rm)


@pytest.mark.parametrize("nlayers,K", [(1, 40), (5, 64), (70, 150)])
def test_select_sphere_batch_equals_sequential(sphere_map, nlayers, K):
    """K strokes in one pass == K successive single strokes (later strokes overwrite)."""
    import torch
    mesh, ref, got = sphere_map
    strokes, labels = synth.sphere_strokes(mesh, K, seed=11 + K, rmin_frac=0.02, rmax_frac=0.2)
    layer_of = (np.arange(K) * 7) % nlayers
    datas = [np.zeros((256, 256), np.uint8) for _ in range(nlayers)]
    masks = [np.zeros((256, 256), bool) for _ in range(nlayers)]
    eds = [np.zeros((256, 256), np.uint8) for _ in range(nlayers)]
    want = np.zeros(nlayers, np.int64)
    for k in range(K):
        L = layer_of[k]
        want[L] += kn.select_sphere(ref["pos"], strokes[k, :3], strokes[k, 3], datas[L], masks[L], eds[L], labels[k])
    mk = lambda dt: [torch.zeros((256, 256), dtype=dt, device="cuda") for _ in range(nlayers)]
    gd, gm, ge = mk(torch.uint8), mk(torch.bool), mk(torch.uint8)
    batch = nat.StrokeBatch(gd, gm, ge, "cuda").upload(strokes, layer_of, labels)
    nat.select_sphere_batch(got["pos"], batch)
    assert np.array_equal(batch.counts.cpu().numpy(), want)
    for L in range(nlayers):
        assert np.array_equal(gd[L].cpu().numpy(), datas[L]), L
        assert np.array_equal(gm[L].cpu().numpy(), masks[L]) and np.array_equal(ge[L].cpu().numpy(), eds[L])


def test_tile_boxes_bound_the_positions(sphere_map):
    """Boxes of the 128 x 4-texel tiles: exact min / max of the covered positions, lo > hi when a
    tile has no covered texel."""
    _, ref, got = sphere_map
    tiles = nat.tile_boxes(got["pos"])
    assert tiles is not None and tiles.boxes.shape == (2 * 64, 8)
    boxes = tiles.boxes.cpu().numpy()
    pos = ref["pos"]
    for ty in range(64):
        for tx in range(2):
            blk = pos[:, 4 * ty: 4 * ty + 4, 128 * tx: 128 * tx + 128].reshape(3, -1)
            b = boxes[ty * 2 + tx]
            if np.isnan(blk[0]).all():
                assert b[0] > b[4]
            else:
                assert np.array_equal(b[0:3], np.nanmin(blk, axis=1)) and np.array_equal(b[4:7], np.nanmax(blk, axis=1))
    assert nat.tile_boxes(got["pos"][:, :, :200].contiguous()) is None          # width % 128 != 0: no culling


@pytest.mark.parametrize("kind,value", [(np.uint8, 9), (np.int16, -5), (np.uint32, 77777)])
def test_select_sphere_culled_bit_exact(sphere_map, kind, value):
    """Footprint-culled brush == oracle (planes and count), incl. a brush that misses everything, one
    that covers everything, a zero radius on a surface point and ragged slab heights."""
    _, ref, got = sphere_map
    rng = np.random.default_rng(5)
    onpoint = tuple(float(v) for v in ref["pos"][:, 130, 70])
    assert not np.isnan(onpoint[0])
    for rows in (256, 255, 3):
        pos_ref = np.ascontiguousarray(ref["pos"][:, :rows])
        pos_dev = got["pos"][:, :rows].contiguous()
        tiles = nat.tile_boxes(pos_dev)
        for center, radius in (((0.0, 0.0, 1.0), 0.25), ((0.6, -0.5, 0.3), 0.6), ((5.0, 5.0, 5.0), 0.1),
                               ((0, 0, 0), 2.0), (onpoint, 0.0), ((0.0, 0.0, 1.0), 1e-3)):
            data0 = rng.integers(0, 4, size=(rows, 256)).astype(kind)
            mask0 = rng.random((rows, 256)) < 0.2
            ed0 = (rng.random((rows, 256)) < 0.1).astype(np.uint8)
            rd, rm, re = data0.copy(), mask0.copy(), ed0.copy()
            want = kn.select_sphere(pos_ref, center, radius, rd, rm, re, value)
            d, m, e = _dev(data0), _dev(mask0), _dev(ed0)
            assert nat.select_sphere(pos_dev, center, radius, d, m, e, value, tiles=tiles) == want
            assert np.array_equal(_bits(_host(d)), _bits(rd))
            assert np.array_equal(m.cpu().numpy(), rm) and np.array_equal(e.cpu().numpy(), re)


def test_select_sphere_degenerate_strokes(sphere_map):
    """NaN / infinite / negative radii and a NaN centre: streamed and culled kernels agree with the
    oracle (NaN never hits, an infinite radius hits every covered texel, r enters only as r*r)."""
    _, ref, got = sphere_map
    tiles = nat.tile_boxes(got["pos"])
    covered = int((ref["tri_id"] >= 0).sum())
    for center, radius in (((0.0, 0.0, 1.0), float("nan")), ((0.0, 0.0, 1.0), float("inf")), ((0.0, 0.0, 1.0), -0.3),
                           ((float("nan"), 0.0, 1.0), 0.5), ((0.0, 0.0, 1.0), 0.0)):
        rd = np.zeros((256, 256), np.uint8); rm = np.zeros((256, 256), bool); re = np.zeros((256, 256), np.uint8)
        want = kn.select_sphere(ref["pos"], center, radius, rd, rm, re, 5)
        for tl in (None, tiles):
            d, m, e = _dev(np.zeros((256, 256), np.uint8)), _dev(np.zeros((256, 256), bool)), _dev(np.zeros((256, 256), np.uint8))
            assert nat.select_sphere(got["pos"], center, radius, d, m, e, 5, tiles=tl) == want
            assert np.array_equal(d.cpu().numpy(), rd) and np.array_equal(m.cpu().numpy(), rm)
        if radius == float("inf"):
            assert want == covered
        if radius != radius or center[0] != center[0]:
            assert want == 0
    # an empty batch is a no-op
    import torch
    gd = [torch.zeros((256, 256), dtype=torch.uint8, device="cuda")]
    gm = [torch.zeros((256, 256), dtype=torch.bool, device="cuda")]
    ge = [torch.zeros((256, 256), dtype=torch.uint8, device="cuda")]
    batch = nat.StrokeBatch(gd, gm, ge, "cuda").upload(np.zeros((0, 4)), np.zeros(0, np.int64), np.zeros(0, np.uint8))
    nat.select_sphere_batch(got["pos"], batch, tiles=tiles)
    nat.select_sphere_batch(got["pos"], batch)
    assert int(batch.counts.sum()) == 0 and not bool(gm[0].any())


@pytest.mark.parametrize("nlayers,K", [(1, 40), (5, 64), (70, 150)])
def test_select_sphere_batch_culled_equals_sequential(sphere_map, nlayers, K):
    import torch
    mesh, ref, got = sphere_map
    strokes, labels = synth.sphere_strokes(mesh, K, seed=21 + K, rmin_frac=0.005, rmax_frac=0.2)
    layer_of = (np.arange(K) * 7) % nlayers
    datas = [np.zeros((256, 256), np.uint8) for _ in range(nlayers)]
    masks = [np.zeros((256, 256), bool) for _ in range(nlayers)]
    eds = [np.zeros((256, 256), np.uint8) for _ in range(nlayers)]
    want = np.zeros(nlayers, np.int64)
    for k in range(K):
        L = layer_of[k]
        want[L] += kn.select_sphere(ref["pos"], strokes[k, :3], strokes[k, 3], datas[L], masks[L], eds[L], labels[k])
    mk = lambda dt: [torch.zeros((256, 256), dtype=dt, device="cuda") for _ in range(nlayers)]
    gd, gm, ge = mk(torch.uint8), mk(torch.bool), mk(torch.uint8)
    batch = nat.StrokeBatch(gd, gm, ge, "cuda").upload(strokes, layer_of, labels)
    nat.select_sphere_batch(got["pos"], batch, tiles=nat.tile_boxes(got["pos"]))
    assert np.array_equal(batch.counts.cpu().numpy(), want)
    for L in range(nlayers):
        assert np.array_equal(gd[L].cpu().numpy(), datas[L]), L
        assert np.array_equal(gm[L].cpu().numpy(), masks[L]) and np.array_equal(ge[L].cpu().numpy(), eds[L])


@pytest.mark.parametrize("akind", [np.float32, np.float16, np.uint8, np.int8, np.int16, np.int32, np.uint32])
def test_select_threshold_bit_exact(akind):
    rng = np.random.default_rng(6)
    h, w = 61, 83                                             # odd sizes: vector body + scalar tail
    if np.issubdtype(akind, np.floating):
        attr = rng.normal(size=(h, w)).astype(akind)
        attr[rng.random((h, w)) < 0.05] = np.nan
        lo, hi = -0.3, 0.7
    else:
        info = np.iinfo(akind)
        attr = rng.integers(max(info.min, -1000), min(info.max, 1000) + 1, size=(h, w)).astype(akind)
        lo, hi = 3.0, 90.0
    for valid in (None, (rng.random((h, w)) < 0.7).astype(np.uint8)):
        rd = np.zeros((h, w), np.int16); rm = np.zeros((h, w), bool); re = np.zeros((h, w), np.uint8)
        want = kn.select_threshold(attr, valid, lo, hi, rd, rm, re, -2)
        d, m, e = _dev(rd * 0), _dev(rm & False), _dev(re * 0)
        got = nat.select_threshold(_dev(attr), None if valid is None else _dev(valid), lo, hi, d, m, e, -2)
        assert got == want
        assert np.array_equal(d.cpu().numpy(), rd) and np.array_equal(m.cpu().numpy(), rm)
        assert np.array_equal(e.cpu().numpy(), re)


def test_select_threshold_rounding_edges():
    """The kernel compares in the attribute's own domain against inward-rounded thresholds; that
    must equal the float64 definition exactly at the representability edges."""
    f = np.float32
    lo, hi = 0.1, 0.7                                         # neither is a float32
    edge = [f(lo), np.nextafter(f(lo), f(1)), np.nextafter(f(lo), f(-1)), f(hi), np.nextafter(f(hi), f(1)),
            np.nextafter(f(hi), f(-1)), f(np.inf), f(-np.inf), f(np.nan), f(0.0), f(-0.0), f(3e38), f(1e-45)]
    cases = [(lo, hi), (-np.inf, np.inf), (1e39, np.inf), (-np.inf, -1e39), (0.0, 0.0), (float(f(lo)), float(f(hi))),
             (0.7, 0.1), (np.nan, 1.0), (-1e-46, 1e-46), (2.5, 1e300)]
    attr32 = np.resize(np.array(edge, f), 64).reshape(4, 16)
    attr16 = attr32.astype(np.float16)
    ints = np.resize(np.array([-3, -2, -1, 0, 1, 2, 3, 100, -100], np.int32), 64).reshape(4, 16)
    int_cases = [(-2.5, 2.5), (-2.0, 2.0), (-1e30, 1e30), (2.0000001, 2.9999), (3.0, 3.0), (1e19, 1e20), (-1e20, -1e19)]
    for attr, cs in ((attr32, cases), (attr16, cases), (ints, int_cases), (ints.astype(np.int8), int_cases),
                     (np.abs(ints).astype(np.uint32), int_cases)):
        for a, b in cs:
            rd = np.zeros(attr.shape, np.uint8); rm = np.zeros(attr.shape, bool); re = np.zeros(attr.shape, np.uint8)
            want = kn.select_threshold(attr, None, a, b, rd, rm, re, 1)
            d, m, e = _dev(rd * 0), _dev(rm & False), _dev(re * 0)
            assert nat.select_threshold(_dev(attr), None, a, b, d, m, e, 1) == want, (attr.dtype, a, b)
            assert np.array_equal(m.cpu().numpy(), rm), (attr.dtype, a, b)


@pytest.mark.parametrize("kind", [None, np.uint8, np.int16, np.float32, np.uint32])
@pytest.mark.parametrize("op", ["union", "intersection", "difference", "masking"])
def test_layer_op_bit_exact(kind, op):
    rng = np.random.default_rng(8)
    n = 16 * 1000 + 13                                        # vector body + tail
    ma = (rng.random(n) < 0.4).astype(np.uint8) * rng.integers(1, 255, n).astype(np.uint8)   # any non-zero = true
    mb = (rng.random(n) < 0.5).astype(np.uint8)
    da = db = None
    if kind is not None:
        da = rng.integers(0, 100, n).astype(kind)
        db = rng.integers(0, 100, n).astype(kind)
    rc = None if kind is None else np.empty(n, kind)
    rmc = np.empty(n, np.uint8)
    kn.layer_op(op, da, ma, db, mb, rc, rmc)
    gd = None if kind is None else _dev(np.zeros(n, kind))
    gm = _dev(np.zeros(n, np.uint8))
    nat.layer_op(op, None if kind is None else _dev(da), _dev(ma),
                 None if (kind is None or op == "masking") else _dev(db), _dev(mb), gd, gm)
    assert np.array_equal(gm.cpu().numpy(), rmc)
    if kind is not None:
        assert np.array_equal(_bits(_host(gd)), _bits(rc))
    # in place: output aliases A
    if kind is not None:
        a_d, a_m = _dev(da), _dev(ma)
        nat.layer_op(op, a_d, a_m, _dev(db), _dev(mb), a_d, a_m)
        assert np.array_equal(_bits(_host(a_d)), _bits(rc)) and np.array_equal(a_m.cpu().numpy(), rmc)


@pytest.mark.parametrize("kind", [None, np.uint8, np.uint32])
def test_layer_chain_equals_sequential_ops(kind):
    """C3 chain ((L0 u L1) n L2) \\ L3 ... over 8 layers, fused vs step-by-step oracle."""
    rng = np.random.default_rng(10)
    n = 16 * 700 + 5
    N = 8
    ops = ["union", "intersection", "difference", "union", "masking", "difference", "union"]
    masks = [(rng.random(n) < 0.45).astype(np.uint8) for _ in range(N)]
    datas = [None] * N if kind is None else [rng.integers(1, 200, n).astype(kind) for _ in range(N)]
    cd = None if kind is None else datas[0].copy()
    cm = masks[0].copy()
    if kind is not None:
        cd[cm == 0] = 0
        cm = (cm != 0).astype(np.uint8)
    for j in range(1, N):
        nd = None if kind is None else np.empty(n, kind)
        nm = np.empty(n, np.uint8)
        kn.layer_op(ops[j - 1], cd, cm, datas[j], masks[j], nd, nm)
        cd, cm = nd, nm
    gd = None if kind is None else _dev(np.zeros(n, kind))
    gm = _dev(np.zeros(n, np.uint8))
    nat.layer_chain(None if kind is None else [_dev(d) for d in datas], [_dev(m) for m in masks], [None] + ops, gd, gm)
    assert np.array_equal(gm.cpu().numpy(), cm)
    if kind is not None:
        assert np.array_equal(_bits(_host(gd)), _bits(cd))


@pytest.mark.parametrize("seed", range(10))
def test_layer_chain_lazy_random_sequences(seed):
    """Chains of 3..8 layers with 1-, 2- or 4-byte data take the lazy-data kernel: random operator sequences, sparse /
    dense / coherent masks, mask bytes other than 0 / 1 (any non-zero byte is valid), ragged length
    (scalar tail), and the output aliasing the first operand -- fused result == step-by-step oracle."""
    rng = np.random.default_rng(500 + seed)
    n = 16 * int(rng.integers(50, 900)) + int(rng.integers(0, 16))
    N = int(rng.integers(3, 9))
    kind = (np.uint8, np.int8, np.int16, np.uint32, np.float32)[seed % 5]
    ops = [str(rng.choice(["union", "intersection", "difference", "masking"])) for _ in range(N - 1)]
    masks = []
    for k in range(N):
        p = float(rng.choice([0.02, 0.3, 0.9]))
        if rng.random() < 0.5:                                   # coherent runs
            m = np.repeat(rng.random(n // 40 + 1) < p, 40)[:n]
        else:
            m = rng.random(n) < p
        m = m.astype(np.uint8) * rng.choice(np.array([1, 1, 1, 2, 255], np.uint8), size=n)
        masks.append(m)
    datas = [rng.integers(-100 if kind in (np.int8, np.int16, np.float32) else 1, 100, n).astype(kind) for _ in range(N)]
    cd, cm = datas[0].copy(), (masks[0] != 0).astype(np.uint8)
    cd[cm == 0] = 0
    for j in range(1, N):
        nd, nm = np.empty(n, kind), np.empty(n, np.uint8)
        kn.layer_op(ops[j - 1], cd, cm, datas[j], masks[j], nd, nm)
        cd, cm = nd, nm
    d_dev, m_dev = [_dev(d) for d in datas], [_dev(m) for m in masks]
    gd, gm = _dev(np.zeros(n, kind)), _dev(np.zeros(n, np.uint8))
    for lazy in (True, False):                                   # lazy-data kernel and the streaming (eager) kernel
        gd.zero_(); gm.zero_()
        nat.layer_chain(d_dev, m_dev, [None] + ops, gd, gm, lazy=lazy)
        assert np.array_equal(gm.cpu().numpy(), cm) and np.array_equal(_bits(_host(gd)), _bits(cd)), (ops, lazy)
    # in place: the result overwrites layer 0
    nat.layer_chain(d_dev, m_dev, [None] + ops, d_dev[0], m_dev[0])
    assert np.array_equal(m_dev[0].cpu().numpy(), cm) and np.array_equal(_bits(_host(d_dev[0])), _bits(cd)), ops


@pytest.mark.parametrize("L", [1, 3, 8, 13, 64])
def test_layer_area_matches_oracle(sphere_map, L):
    _, ref, got = sphere_map
    rng = np.random.default_rng(12 + L)
    masks = [(rng.random((256, 256)) < rng.uniform(0.05, 0.9)).astype(np.uint8) for _ in range(L)]
    sums, counts = nat.layer_area(got["area"], [_dev(m) for m in masks])
    for l in range(L):
        a, c = kn.layer_area(ref["area"], masks[l])
        assert counts[l] == c
        assert abs(sums[l] - a) <= 1e-10 * max(abs(a), 1e-300)


def test_sphere_area_close_to_analytic(sphere_map):
    """Whole-atlas area of the unit icosphere ~= mesh area (texel sampling error only)."""
    mesh, ref, got = sphere_map
    from paper_2501_14807_b200 import mesh_surface_area
    full = (ref["tri_id"] >= 0).astype(np.uint8)
    sums, _ = nat.layer_area(got["area"], [_dev(full)])
    assert abs(sums[0] - mesh_surface_area(mesh)) / mesh_surface_area(mesh) < 0.05
    assert abs(kn.mesh_surface_area(mesh.tri_pos()) - mesh_surface_area(mesh)) < 1e-12


def test_label_area_and_stats(sphere_map):
    _, ref, got = sphere_map
    rng = np.random.default_rng(14)
    data = np.repeat(np.repeat(rng.integers(0, 256, size=(32, 32)), 8, 0), 8, 1).astype(np.uint8)
    mask = (rng.random((256, 256)) < 0.8).astype(np.uint8)
    want_s, want_c = kn.label_area(ref["area"], data, mask)
    s, c = nat.label_area(got["area"], _dev(data), _dev(mask))
    assert np.array_equal(c, want_c)
    assert np.allclose(s, want_s, rtol=1e-10, atol=0)
    for akind in (np.float32, np.int16, np.uint8, np.float16):
        attr = (rng.normal(size=(256, 256)) * 50).astype(akind)
        wc, ws, wmn, wmx = kn.layer_stats(attr, mask)
        gc, gs, gmn, gmx = nat.layer_stats(_dev(attr), _dev(mask))
        assert (gc, gmn, gmx) == (wc, wmn, wmx) and abs(gs - ws) <= 1e-9 * max(1.0, abs(ws))


@pytest.mark.parametrize("akind", [np.uint8, np.int8, np.int16, np.int32, np.uint32, np.float16, np.float32])
def test_layer_stats_all_kinds_ragged_and_unaligned(akind):
    """Vector path (16 texels per step), its scalar tail (n % 16 != 0), planes at odd offsets, an
    empty mask (count 0, min = +inf, max = -inf like the oracle) and a single valid texel."""
    import torch
    rng = np.random.default_rng(15)
    for n, off in ((16 * 37 + 5, 0), (4099, 3), (7, 0)):
        raw = (rng.normal(size=n + off) * 40).astype(akind)
        rmask = (rng.random(n + off) < 0.6).astype(np.uint8)
        attr, mask = raw[off:], rmask[off:]
        d_attr, d_mask = _dev(raw)[off:], _dev(rmask)[off:]
        for m_np, m_dev in ((mask, d_mask), (np.zeros_like(mask), torch.zeros_like(d_mask))):
            want = kn.layer_stats(np.ascontiguousarray(attr), np.ascontiguousarray(m_np))
            gc, gs, gmn, gmx = nat.layer_stats(d_attr, m_dev)
            assert (gc, gmn, gmx) == (want[0], want[2], want[3])
            assert abs(gs - want[1]) <= 1e-9 * max(1.0, abs(want[1]))
    one = np.zeros(64, np.uint8); one[37] = 1
    a = np.arange(64).astype(akind)
    assert nat.layer_stats(_dev(a), _dev(one))[0::2] == (1, 37.0) and nat.layer_stats(_dev(a), _dev(one))[3] == 37.0


def test_outline_and_padding_known_answers():
    """10x10 island in 64x64, thickness 1 -> 44 outline texels."""
    import torch
    cov = np.zeros((64, 64), np.uint8)
    cov[20:30, 30:40] = 1
    out = nat.outline_mask(_dev(cov), 1)
    assert int(out.sum().item()) == 44 and np.array_equal(out.cpu().numpy(), kn.outline(cov, 1))
    assert int(nat.outline_mask(_dev(np.ones((64, 64), np.uint8)), 1).sum().item()) == 0
    assert int(nat.outline_mask(_dev(np.zeros((64, 64), np.uint8)), 1).sum().item()) == 0
    edited = np.zeros((64, 64), np.uint8)
    edited[29, 35] = 1                                       # adjacent to the island border
    data = torch.zeros((64, 64), dtype=torch.int16, device="cuda")
    mask = torch.zeros((64, 64), dtype=torch.bool, device="cuda")
    n = nat.apply_padding(out, _dev(edited), 1, data, mask, 42)
    rd = np.zeros((64, 64), np.int16); rm = np.zeros((64, 64), bool)
    assert n == kn.padding(kn.outline(cov, 1), edited, 1, rd, rm, 42) == 3
    assert np.array_equal(data.cpu().numpy(), rd) and np.array_equal(mask.cpu().numpy(), rm)
    assert nat.apply_padding(out, _dev(edited), 0, data, mask, 42) == 0


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("r", [1, 2, 5])
def test_outline_and_padding_random(seed, r):
    """randomized island layouts, padded set == outline within Chebyshev r of edited."""
    import torch
    rng = np.random.default_rng(100 + seed)
    # odd widths take the generic kernel, multiples of 16 the streaming kernel (radius <= 4)
    h, w = 64 + seed, (70 + 3 * seed) if seed % 2 else (64 + 16 * seed)
    cov = (rng.random((h, w)) < 0.03).astype(np.uint8)
    cov = (kn.outline(cov, 2) | cov).astype(np.uint8)        # blobby islands
    ref_out = kn.outline(cov, r)
    got_out = nat.outline_mask(_dev(cov), r)
    assert np.array_equal(got_out.cpu().numpy(), ref_out)
    assert not (ref_out & cov).any()
    edited = ((rng.random((h, w)) < 0.05) & (cov != 0)).astype(np.uint8)
    rd = np.zeros((h, w), np.uint8); rm = np.zeros((h, w), bool)
    want = kn.padding(ref_out, edited, r, rd, rm, 9)
    d = torch.zeros((h, w), dtype=torch.uint8, device="cuda"); m = torch.zeros((h, w), dtype=torch.bool, device="cuda")
    assert nat.apply_padding(got_out, _dev(edited), r, d, m, 9) == want
    assert np.array_equal(d.cpu().numpy(), rd) and np.array_equal(m.cpu().numpy(), rm)
    # row slabs with halo == full
    parts = []
    for r0, r1 in ((0, 20), (20, h)):
        i0, i1 = max(0, r0 - r), min(h, r1 + r)
        parts.append(nat.outline_mask(_dev(cov[i0:i1]), r, in_row0=i0, out_row0=r0, out_rows=r1 - r0).cpu().numpy())
    assert np.array_equal(np.concatenate(parts), ref_out)


def test_c_abi_argument_validation():
    """Return codes of the C ABI for arguments the kernels cannot take (ML_ERR_ARG = 1 with a message
    in ml_last_error); nothing is launched and no plane is touched."""
    import ctypes as C
    import torch
    L = nat.lib()
    z = torch.zeros((8, 200), dtype=torch.uint8, device="cuda")
    pos = torch.zeros((3, 8, 200), dtype=torch.float32, device="cuda")
    p = lambda t: C.c_void_p(t.data_ptr())
    none = C.c_void_p(0)
    # culled brushes need width % 128 == 0, the boxes and the scratch
    assert L.ml_tile_count(200, 8) == 0 and L.ml_tile_count(256, 9) == 2 * 3
    assert L.ml_tile_workspace_bytes(200, 8) == 16
    assert L.ml_surface_tile_boxes(p(pos), 1600, 200, 8, p(z), none) == 1
    assert b"128" in L.ml_last_error()
    assert L.ml_select_sphere_tiles(p(pos), 1600, 200, 8, none, none, 0, 0.0, 0.0, 0.0, 1.0, p(z), 1, 1, p(z), p(z), none, none) == 1
    pos2 = torch.zeros((3, 8, 256), dtype=torch.float32, device="cuda")
    z2 = torch.zeros((8, 256), dtype=torch.uint8, device="cuda")
    assert L.ml_select_sphere_tiles(p(pos2), 2048, 256, 8, none, none, 0, 0.0, 0.0, 0.0, 1.0, p(z2), 1, 1, p(z2), p(z2), none, none) == 1
    assert b"boxes" in L.ml_last_error()
    boxes = torch.zeros((4, 8), dtype=torch.float32, device="cuda")
    assert L.ml_select_sphere_tiles(p(pos2), 2048, 256, 8, p(boxes), none, 0, 0.0, 0.0, 0.0, 1.0, p(z2), 1, 1, p(z2), p(z2), none, none) == 1
    assert b"scratch" in L.ml_last_error()
    # element size / record buffers / padding tiles
    assert L.ml_select_sphere(p(pos), 1600, 1600, 0.0, 0.0, 0.0, 1.0, p(z), 3, 1, p(z), p(z), none, none) == 1
    assert L.ml_tea_prepare(p(pos), p(pos), 7, 10, p(z), 10 ** 6, none) == 1                 # buffer too small comes first
    big = torch.zeros(int(L.ml_tea_rec_bytes(10)), dtype=torch.uint8, device="cuda")
    assert L.ml_tea_prepare(p(pos), p(pos), 7, 10, p(big), big.numel(), none) == 1           # unknown dtype code
    assert L.ml_tea_prepare(p(pos), p(pos), 7, 0, none, 0, none) == 0                        # no triangles: no-op
    assert L.ml_apply_padding_tiles(p(z), p(z), 200, 8, 1, none, p(z), 1, 1, p(z), none, none) == 1
    assert L.ml_apply_padding_tiles(p(z2), p(z2), 256, 8, 9, p(z2), p(z2), 1, 1, p(z2), none, none) == 1   # radius > 4
    assert L.ml_apply_padding_tiles(p(z2), p(z2), 256, 8, 0, none, p(z2), 1, 1, p(z2), none, none) == 0    # radius 0: no-op
    assert L.ml_surface_resolve(none, none, none, 1, 4, 256, 0, 8, none, none, none, none, none, none, 0, none) == 1
    torch.cuda.synchronize()
    assert not bool(z.any()) and not bool(z2.any())


def test_classification_from_bounds_is_a_superset():
    """ml_tea_classify_recs (16-byte outward-rounded bounds) must keep every triangle ml_tea_classify
    keeps -- on random clip-space triangles incl. mixed signs of w, w == 0, NaN / inf coordinates, huge
    and tiny magnitudes, and random tool maps (negative scales, degenerate zero scale)."""
    import ctypes as C
    import torch
    L = nat.lib()
    rng = np.random.default_rng(77)
    T = 20000
    clip = np.empty((T, 3, 4))
    w = rng.uniform(0.05, 4.0, size=(T, 3)) * np.exp(rng.uniform(-6, 6, size=(T, 1)))
    w[rng.random((T, 3)) < 0.1] *= -1.0
    w[rng.random((T, 3)) < 0.01] = 0.0
    clip[..., 3] = w
    clip[..., 0] = rng.uniform(-3, 3, size=(T, 3)) * np.abs(w) + rng.normal(size=(T, 3)) * 1e-3
    clip[..., 1] = rng.uniform(-3, 3, size=(T, 3)) * np.abs(w)
    clip[..., 2] = rng.uniform(-1, 1, size=(T, 3)) * np.abs(w)
    bad = rng.random(T) < 0.01
    clip[bad, rng.integers(0, 3, bad.sum()), rng.integers(0, 4, bad.sum())] = rng.choice([np.nan, np.inf, -np.inf], bad.sum())
    xy = rng.uniform(0, 256, size=(T, 3, 2))
    depth = torch.ones((64, 64), dtype=torch.float32, device="cuda")
    shape = torch.ones((8, 8), dtype=torch.uint8, device="cuda")
    for dt in (np.float64, np.float32):
        d_clip, d_xy = _dev(clip.astype(dt)), _dev(xy.astype(dt))
        code = nat.ML_F64 if dt == np.float64 else nat.ML_F32
        recs = nat.tea_prepare(d_xy, d_clip)
        nw = (T + 31) // 32
        for k in range(12):
            sfx, sfy = rng.uniform(-20, 20, size=2) * (0.0 if k == 11 else 1.0)
            bx, by = rng.uniform(-8, 8, size=2)
            p = nat._tea_params(64.0, 64.0, depth, 1e-4, sfx, sfy, bx, by, shape)
            f0 = torch.zeros(nw, dtype=torch.int32, device="cuda")
            f1 = torch.zeros(nw, dtype=torch.int32, device="cuda")
            assert L.ml_tea_classify(C.c_void_p(d_clip.data_ptr()), code, T, C.byref(p), C.c_void_p(f0.data_ptr()), None,
                                     256, 256, 0, 256, None, None) == 0
            assert L.ml_tea_classify_recs(C.c_void_p(recs.data_ptr()), code, T, C.byref(p), C.c_void_p(f1.data_ptr()), None,
                                          256, 256, 0, 256, None, None) == 0
            a, b = f0.cpu().numpy().view(np.uint32), f1.cpu().numpy().view(np.uint32)
            assert not (a & ~b).any(), (dt, k)
            kept0 = int(np.unpackbits(a.view(np.uint8)).sum()); kept1 = int(np.unpackbits(b.view(np.uint8)).sum())
            assert kept0 <= kept1 <= kept0 + max(50, kept0 // 50)           # and not much looser


@pytest.mark.parametrize("kind,value", [(np.uint8, 9), (np.int16, -5), (np.float32, 0.25)])
def test_select_threshold_culled_bit_exact(sphere_map, kind, value):
    """Tile-range culled threshold on a float32 attribute with NaN holes (the surface map's z plane)
    == oracle: windows that miss everything, hit everything, sit on exact attribute values, have
    +-inf ends, are empty (lo > hi) or NaN; with and without a valid plane; ragged slab heights."""
    _, ref, got = sphere_map
    rng = np.random.default_rng(8)
    z_ref = np.ascontiguousarray(ref["pos"][2])
    some = float(z_ref[130, 70])
    assert some == some
    for rows in (256, 255, 6):
        attr_ref = np.ascontiguousarray(z_ref[:rows])
        attr_dev = got["pos"][2][:rows].contiguous()
        tiles = nat.attr_tiles(attr_dev)
        assert tiles is not None
        ranges = tiles.ranges.cpu().numpy()
        blk = attr_ref[:4, :128]
        if not np.isnan(blk).all():
            assert ranges[0, 0] == np.nanmin(blk) and ranges[0, 1] == np.nanmax(blk)
        valid_np = (rng.random((rows, 256)) < 0.7).astype(np.uint8)
        for lo, hi in ((-0.2, 0.3), (5.0, 6.0), (-9.0, 9.0), (some, some), (-np.inf, 0.0), (0.5, np.inf), (0.3, -0.3),
                       (np.nan, 1.0), (np.nextafter(some, 2.0), 0.99)):
            for valid in (None, valid_np):
                data0 = rng.integers(0, 4, size=(rows, 256)).astype(kind)
                mask0 = rng.random((rows, 256)) < 0.2
                ed0 = (rng.random((rows, 256)) < 0.1).astype(np.uint8)
                rd, rm, re = data0.copy(), mask0.copy(), ed0.copy()
                want = kn.select_threshold(attr_ref, valid, lo, hi, rd, rm, re, value)
                d, m, e = _dev(data0), _dev(mask0), _dev(ed0)
                assert nat.select_threshold(attr_dev, None if valid is None else _dev(valid), lo, hi, d, m, e, value,
                                            tiles=tiles) == want, (rows, lo, hi)
                assert np.array_equal(_bits(_host(d)), _bits(rd))
                assert np.array_equal(m.cpu().numpy(), rm) and np.array_equal(e.cpu().numpy(), re)
    assert nat.attr_tiles(got["pos"][2][:, :200].contiguous()) is None and nat.attr_tiles(got["tri_id"]) is None


@pytest.mark.parametrize("L", [1, 2, 3, 8])
def test_layer_area_counts_exact_over_many_ring_rounds(L):
    """Regression for a cross-proxy race in the bulk-copy ring (csrc/bulk.cuh): with small stages (one or two mask
    planes per group -> 4-8 KB stages recycled thousands of times) consumers read bytes of the NEXT round unless
    they fence the async proxy before releasing a stage.  Texel counts over 16.8 M texels must be exact, every time."""
    import torch
    N = 4096 * 4096
    g = torch.Generator(device="cuda").manual_seed(7 + L)
    area = torch.rand(N, device="cuda", dtype=torch.float32, generator=g)
    masks = [(torch.rand(N, device="cuda", generator=g) < 0.3).to(torch.uint8) for _ in range(L)]
    want_c = [int(m.sum()) for m in masks]
    want_s = [float((area.double() * m.double()).sum()) for m in masks]
    for rep in range(5):
        sums = torch.zeros(L, dtype=torch.float64, device="cuda")
        cnts = torch.zeros(L, dtype=torch.int64, device="cuda")
        nat.layer_area(area.view(1, N), [m.view(1, N) for m in masks], sums=sums, counts=cnts)
        assert cnts.tolist() == want_c
        assert all(abs(a - b) <= 1e-12 * b for a, b in zip(sums.tolist(), want_s))
