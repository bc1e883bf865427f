"""The bulk-copy ring kernels (csrc/bulk.cuh: cp.async.bulk + mbarrier; threshold, area, TPA padding, TEA id stream)
only take over above a size threshold, so the small parity suites run the register forms.  Here: mid-size planes
with RAGGED sizes (texel counts that are no multiple of a 16-texel vector, of a 512-texel warp tile or of a ring
chunk, so the last chunk of every block is partial and the scalar tails run), every attribute kind, every layer
element size, with and without a valid plane, each against the oracle AND against the register form of the same
kernel (environment switch), bit for bit."""
import os
import subprocess
import sys

import numpy as np
import pytest

import helpers
from oracle import kn
from paper_2501_14807_b200 import _native as nat
from paper_2501_14807_b200 import synth
import paper_2501_14807_b200 as ml

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _dev(a):
    import torch
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        return torch.from_numpy(a.view(np.int32)).cuda().view(torch.uint32)
    if a.dtype == np.uint16:
        return torch.from_numpy(a.view(np.int16)).cuda().view(torch.uint16)
    return torch.from_numpy(a).cuda()


def _host(t):
    import torch
    if t.dtype == torch.uint32:
        return t.view(torch.int32).cpu().numpy().view(np.uint32)
    return t.cpu().numpy()


@pytest.mark.parametrize("akind", [np.float32, np.float16, np.uint8, np.int8, np.int16, np.int32, np.uint32])
@pytest.mark.parametrize("dkind,value", [(np.uint8, 201), (np.int16, -2), (np.float32, 1.5)])
def test_threshold_bulk_ragged_all_kinds(akind, dkind, value):
    rng = np.random.default_rng(11)
    h, w = 401, 403                                           # 161,603 texels: 3 tail texels, partial warp tile and chunk
    yy, xx = np.mgrid[0:h, 0:w]
    field = np.sin(xx / 17.0) * np.cos(yy / 23.0) + 0.15 * rng.normal(size=(h, w))       # coherent band with ragged edges
    if np.issubdtype(akind, np.floating):
        attr = field.astype(akind)
        attr[rng.random((h, w)) < 0.02] = np.nan
        lo, hi = -0.2, 0.35
    else:
        info = np.iinfo(akind)
        attr = np.clip(field * 100, max(info.min, -120), min(info.max, 120)).astype(akind)
        lo, hi = 3.0, 60.0
    for valid in (None, (rng.random((h, w)) < 0.8).astype(np.uint8)):
        d0 = rng.integers(0, 5, size=(h, w)).astype(dkind)
        m0 = rng.random((h, w)) < 0.2
        e0 = (rng.random((h, w)) < 0.1).astype(np.uint8) * rng.integers(1, 4, size=(h, w)).astype(np.uint8)   # bytes 0..3
        rd, rm, re = d0.copy(), m0.copy(), e0.copy()
        want = kn.select_threshold(attr, valid, lo, hi, rd, rm, re, value)
        d, m, e = _dev(d0), _dev(m0), _dev(e0)
        got = nat.select_threshold(_dev(attr), None if valid is None else _dev(valid), lo, hi, d, m, e, value)
        assert got == want and want > 0
        assert np.array_equal(_host(d).view(np.uint8), rd.view(np.uint8))
        assert np.array_equal(m.cpu().numpy(), rm) and np.array_equal(e.cpu().numpy(), re)


@pytest.mark.parametrize("L", [1, 2, 3, 5, 8, 11])
def test_area_bulk_ragged(L):
    import torch
    rng = np.random.default_rng(5 + L)
    n = 70_003                                                # >= 4 chunks of 4096, 3 tail texels
    area = rng.random(n).astype(np.float32)
    masks = []
    for k in range(L):
        m = (rng.random(n) < 0.35).astype(np.uint8)
        m[1000 * k:1000 * k + 4096] = 1                       # runs of fully set words
        m[20000:26000] = 0                                    # a stretch where every mask is empty (area vector skipped)
        if k == 1:
            m[m != 0] = 7                                     # non-{0,1} mask bytes count as set
        masks.append(m)
    sums = torch.zeros(L, dtype=torch.float64, device="cuda")
    cnts = torch.zeros(L, dtype=torch.int64, device="cuda")
    nat.layer_area(_dev(area).view(1, n), [_dev(m).view(1, n) for m in masks], sums=sums, counts=cnts)
    for k in range(L):
        ws, wc = kn.layer_area(area.reshape(1, n), masks[k].reshape(1, n))
        assert int(cnts[k]) == wc
        assert abs(float(sums[k]) - ws) <= 1e-12 * ws


@pytest.mark.parametrize("dkind,value", [(np.uint8, 9), (np.int16, -300), (np.uint32, 3123456789)])
@pytest.mark.parametrize("radius", [1, 3])
def test_padding_bulk_ragged(dkind, value, radius):
    rng = np.random.default_rng(3)
    h, w = 259, 272                                           # width % 16 == 0 (vector path), 70,448 texels = 8.6 chunks
    cov = np.zeros((h, w), np.uint8)
    for _ in range(40):                                       # many small islands: outline vectors all over the plane
        y, x = rng.integers(5, h - 30), rng.integers(5, w - 30)
        cov[y:y + rng.integers(4, 25), x:x + rng.integers(4, 25)] = 1
    outline = kn.outline(cov, 1)
    edited = ((rng.random((h, w)) < 0.05) & (cov != 0)).astype(np.uint8)
    d0 = rng.integers(0, 5, size=(h, w)).astype(dkind)
    m0 = (rng.random((h, w)) < 0.3)
    rd, rm = d0.copy(), m0.copy()
    want = kn.padding(outline, edited, radius, rd, rm, value)
    d, m = _dev(d0), _dev(m0)
    got = nat.apply_padding(_dev(outline), _dev(edited), radius, d, m, value)
    assert got == want and want > 0
    assert np.array_equal(_host(d).view(np.uint8), rd.view(np.uint8)) and np.array_equal(m.cpu().numpy(), rm)


@pytest.mark.parametrize("dkind,value", [(np.uint8, 7), (np.int16, -9), (np.float32, 0.25)])
def test_tea_stream_bulk_with_folded_reset(dkind, value):
    """Whole-atlas TEA (id stream through the ring, EditedAreaMask reset folded in) on an atlas whose texel count is
    no multiple of the 32 KB id chunk, into planes that already hold data and a DIRTY edited plane: == oracle."""
    import torch
    mesh = synth.icosphere_mesh(3)
    A_w, A_h, W = 304, 301, 96                                # 91,504 texels: 11.2 chunks, not a multiple of 4 rows x 128
    cam = synth.default_camera(W, W)
    surf = ml.build_surface_map(mesh, A_w, A_h)
    depth = ml.render_depth(mesh, cam)
    ctx = ml.StrokeContext(mesh, cam, depth, surf)
    layer = ml.create_layer("L", np.dtype(dkind).name, A_w, A_h, pool=ml.TexturePool())
    tool = ml.EditingTool(px=50.0, py=44.0, shape=synth.circle_shape(18), value=value)
    ctx.edited.fill_(3)                                       # stale marks everywhere: the stream must clear all of them
    res = ml.apply_stroke(ctx, tool, layer, cull=False)
    from paper_2501_14807_b200.mesh_core import window_triangles
    xy, zn = window_triangles(mesh, cam)
    d_ref = np.ones((W, W), np.float32)
    kn.raster_depth(xy, zn, d_ref)
    sfx, sfy, bx, by = ml.compute_tool_projection(cam, tool).kernel_factors
    data = np.zeros((A_h, A_w), dkind); mask = np.zeros((A_h, A_w), bool); edited = np.zeros((A_h, A_w), np.uint8)
    tri_xy = mesh.tri_uv_texels(A_w, A_h)
    want = kn.raster_tea(tri_xy, cam.clip_coords(mesh.vertices)[mesh.triangles], float(W), float(W), d_ref, 1e-4, sfx, sfy,
                         bx, by, tool.shape, data, mask, edited, value)
    assert (res.edited_count, res.fragments) == want and want[0] > 0
    assert np.array_equal(_host(layer.data).view(np.uint8), data.view(np.uint8))
    assert np.array_equal(layer.mask.cpu().numpy(), mask)
    assert np.array_equal(ctx.edited.cpu().numpy(), edited)


def test_tea_stream_bulk_with_the_bitmap_in_global_memory():
    """More triangles than the shared-memory bitmap holds beside the ring (> ~1.07 M): the id stream looks the
    classification bits up in global memory (the SMEM = false instantiation).  1,155,200-triangle heightfield on a
    2048^2 atlas, whole-atlas TEA == oracle."""
    import torch
    mesh = synth.heightfield_mesh(760, margin=0.01)
    assert mesh.num_triangles > 1_100_000
    A, W = 2048, 256
    cam = synth.default_camera(W, W, eye=(0.5, 0.5, 1.6), target=(0.5, 0.5, 0.0), fovy=40.0, near=0.2, far=5.0)
    surf = ml.build_surface_map(mesh, A, A)
    depth = ml.render_depth(mesh, cam)
    ctx = ml.StrokeContext(mesh, cam, depth, surf)
    layer = ml.create_layer("L", "uint8", A, A, pool=ml.TexturePool())
    tool = ml.EditingTool(px=120.0, py=131.0, shape=synth.circle_shape(30), value=5)
    res = ml.apply_stroke(ctx, tool, layer, cull=False)
    sfx, sfy, bx, by = ml.compute_tool_projection(cam, tool).kernel_factors
    data = np.zeros((A, A), np.uint8); mask = np.zeros((A, A), bool); edited = np.zeros((A, A), np.uint8)
    want = kn.raster_tea_slab(mesh.tri_uv_texels(A, A), cam.clip_coords(mesh.vertices)[mesh.triangles], float(W), float(W),
                              depth.plane.cpu().numpy(), 1e-4, sfx, sfy, bx, by, tool.shape, data, mask, edited, 5, A, 0,
                              kn.max_threads())
    assert (res.edited_count, res.fragments) == want and want[0] > 0
    assert np.array_equal(layer.data.cpu().numpy(), data) and np.array_equal(layer.mask.cpu().numpy(), mask)
    assert np.array_equal(ctx.edited.cpu().numpy(), edited)


REGISTER_FORMS = {"ML_THR_REGISTER_STREAM": "1", "ML_THR_QUAD_STREAM": "1", "ML_AREA_REGISTER_STREAM": "1",
                  "ML_PAD_REGISTER_STREAM": "1", "ML_TEA_REGISTER_STREAM": "1"}


@pytest.mark.skipif(os.environ.get("ML_THR_REGISTER_STREAM") is not None, reason="already the register-form run")
def test_register_forms_pass_the_same_tests():
    """The register forms stay in the library (unaligned planes, small inputs, A/B timing); the environment switches
    that select them are read once per process, so this re-runs the file in a child process with all of them set."""
    env = dict(os.environ, **REGISTER_FORMS)
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.abspath(__file__), "-x", "-q", "-m", "gpu",
                        "-k", "not register_forms"], capture_output=True, text=True, env=env, cwd=ROOT, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
