"""GPU tests of the SPEC-level surface (pool, layers, stroke pipeline, display, layer files) and
the acceptance criteria that involve the hot path (SPEC.md:603-617 #1, #2, #4, #5, #9)."""
import numpy as np
import pytest

import helpers
import paper_2501_14807_b200 as ml
from oracle import kn
from paper_2501_14807_b200 import _native as nat
from paper_2501_14807_b200 import synth
from paper_2501_14807_b200.mesh_core import window_triangles

pytestmark = pytest.mark.gpu


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# ------------------------------------------------------------------ pool / layers

def test_texture_pool_contract():
    pool = ml.TexturePool(budget_texels=3 * 64 * 64 + 10)
    a = pool.acquire(64, 64, "uint8")
    b = pool.acquire(64, 64, "uint8")
    c = pool.acquire(64, 64, "float32")
    assert len(pool.keys) == 2 and pool.plane_count((64, 64, "uint8")) == 2
    assert not bool(a.tensor.any()) and a.tensor.dtype.is_floating_point is False
    a.tensor.fill_(7)
    a.release()
    a2 = pool.acquire(64, 64, "uint8")
    assert a2.slot == a.slot and not bool(a2.tensor.any())
    with pytest.raises(ml.CapacityExceeded):
        pool.acquire(64, 64, "int16")
    with pytest.raises(ml.TargetMismatch):
        pool.acquire(0, 4, "uint8")
    assert (b.kind, c.kind) == ("uint8", "float32")


def test_create_layer_and_kinds():
    pool = ml.TexturePool()
    for kind in ("int8", "int16", "int32", "uint8", "float16", "float32", "uint32"):
        L = ml.create_layer("k", kind, 40, 24, pool=pool)
        assert L.shape == (24, 40) and L.valid_texels() == 0
    assert (40, 24, "int8") in pool.keys
    with pytest.raises(ml.TargetMismatch):
        ml.create_layer("bad", "complex64", 4, 4, pool=pool)


# ------------------------------------------------------------------ stroke pipeline vs the oracle

def _scene(level=2, atlas=128, window=96):
    mesh = synth.icosphere_mesh(level)
    cam = synth.default_camera(window, window)
    surf = ml.build_surface_map(mesh, atlas, atlas)
    depth = ml.render_depth(mesh, cam)
    return mesh, cam, surf, depth, ml.StrokeContext(mesh, cam, depth, surf)


def _oracle_stroke(mesh, cam, tool, atlas, data, mask, edited, eps=1e-4):
    xy, zn = window_triangles(mesh, cam)
    d = np.ones((cam.height, cam.width), np.float32)
    kn.raster_depth(xy, zn, d)
    sfx, sfy, bx, by = ml.compute_tool_projection(cam, tool).kernel_factors
    return kn.raster_tea(mesh.tri_uv_texels(atlas, atlas), cam.clip_coords(mesh.vertices)[mesh.triangles],
                         float(cam.width), float(cam.height), d, eps, sfx, sfy, bx, by, np.asarray(tool.shape),
                         data, mask, edited, tool.value)


@pytest.mark.parametrize("seed", range(20))
def test_apply_stroke_equals_oracle_random_scenes(seed):              # SPEC.md:605 acceptance #1
    """>= 20 randomised scenes: random camera + tool, edited set == oracle exactly, both TEA kernels."""
    rng = np.random.default_rng(400 + seed)
    mesh = synth.icosphere_mesh(2)
    A, W = 128, int(rng.integers(48, 128))
    eye = rng.normal(size=3)
    eye = eye / np.linalg.norm(eye) * rng.uniform(1.6, 4.0)
    cam = synth.default_camera(W, W, eye=tuple(eye), fovy=float(rng.uniform(30, 70)), near=0.3, far=12.0)
    surf = ml.build_surface_map(mesh, A, A)
    depth = ml.render_depth(mesh, cam)
    ctx = ml.StrokeContext(mesh, cam, depth, surf)
    r = int(rng.integers(3, 30))
    shape = synth.circle_shape(r) if seed % 2 else synth.square_shape(2 * r)
    tool = ml.EditingTool(px=float(rng.uniform(0, W)), py=float(rng.uniform(0, W)), shape=shape, value=int(rng.integers(1, 200)))
    data = np.zeros((A, A), np.uint8); mask = np.zeros((A, A), bool); edited = np.zeros((A, A), np.uint8)
    want = _oracle_stroke(mesh, cam, tool, A, data, mask, edited)
    for direct in (False, True):
        layer = ml.create_layer("L", "uint8", A, A, pool=ml.TexturePool())
        res = ml.apply_stroke(ctx, tool, layer, force_direct=direct)
        assert (res.edited_count, res.fragments) == want
        assert np.array_equal(layer.data.cpu().numpy(), data) and np.array_equal(layer.mask.cpu().numpy(), mask)
        assert np.array_equal(res.edited_mask.cpu().numpy(), edited)
        assert res.transfer_bytes == 64                                              # SPEC.md:609 acceptance #5


@pytest.mark.parametrize("seed", range(6))
def test_strokes_with_camera_inside_the_mesh(seed):
    """Camera INSIDE the sphere with a wide field of view: many triangles have vertices behind the
    camera (w <= 0, mixed signs of w within a triangle), window coordinates far outside the viewport
    and random non-convex tool shapes -- the conservative classification must keep every triangle
    the per-fragment filters could accept.  Culled, streamed and direct kernels == oracle."""
    rng = np.random.default_rng(900 + seed)
    mesh = synth.icosphere_mesh(3)
    A, W = 256, 96
    eye = rng.uniform(-0.4, 0.4, size=3)
    target = eye + rng.normal(size=3)
    cam = synth.default_camera(W, W, eye=tuple(eye), target=tuple(target), fovy=float(rng.uniform(60, 140)), near=0.05, far=4.0)
    surf = ml.build_surface_map(mesh, A, A)
    depth = ml.render_depth(mesh, cam)
    ctx = ml.StrokeContext(mesh, cam, depth, surf)
    shape = (rng.random((int(rng.integers(5, 60)), int(rng.integers(5, 60)))) < 0.6).astype(np.uint8)
    tool = ml.EditingTool(px=float(rng.uniform(-10, W + 10)), py=float(rng.uniform(-10, W + 10)), shape=shape, value=5)
    data = np.zeros((A, A), np.uint8); mask = np.zeros((A, A), bool); edited = np.zeros((A, A), np.uint8)
    want = _oracle_stroke(mesh, cam, tool, A, data, mask, edited)
    pool = ml.TexturePool()
    for mode in ("cull", "stream", "direct"):
        layer = ml.create_layer(mode, "uint8", A, A, pool=pool)
        res = ml.apply_stroke(ctx, tool, layer, cull=(mode == "cull"), force_direct=(mode == "direct"))
        assert (res.edited_count, res.fragments) == want, mode
        assert np.array_equal(layer.data.cpu().numpy(), data) and np.array_equal(res.edited_mask.cpu().numpy(), edited), mode


def test_footprint_culling_sequence_equals_oracle():
    """A sequence of strokes on ONE context: with footprint culling the per-stroke EditedAreaMask
    (cleared only where the previous stroke could have written) and the layer planes must equal
    the oracle after every stroke, and the un-culled / direct paths interleaved in between."""
    import torch
    rng = np.random.default_rng(21)
    mesh = synth.icosphere_mesh(3)
    A, W = 256, 160
    cam = synth.default_camera(W, W)
    surf = ml.build_surface_map(mesh, A, A)
    ctx = ml.StrokeContext(mesh, cam, ml.render_depth(mesh, cam), surf)
    assert ctx.tiles is not None                                      # 256 % 128 == 0 -> culling available
    layer = ml.create_layer("L", "uint8", A, A, pool=ml.TexturePool())
    data = np.zeros((A, A), np.uint8); mask = np.zeros((A, A), bool)
    modes = ["cull", "cull", "cull", "stream", "cull", "direct", "cull", "cull", "stream", "cull", "cull", "cull"]
    for k, mode in enumerate(modes):
        tool = ml.EditingTool(px=float(rng.uniform(30, 130)), py=float(rng.uniform(30, 130)),
                              shape=synth.circle_shape(int(rng.integers(3, 25))), value=k + 1)
        edited = np.zeros((A, A), np.uint8)                           # the oracle's mask is fresh per stroke
        want = _oracle_stroke(mesh, cam, tool, A, data, mask, edited)
        res = ml.apply_stroke(ctx, tool, layer, cull=(mode == "cull"), force_direct=(mode == "direct"))
        assert (res.edited_count, res.fragments) == want, (k, mode)
        assert np.array_equal(res.edited_mask.cpu().numpy(), edited), (k, mode)
        assert np.array_equal(layer.data.cpu().numpy(), data) and np.array_equal(layer.mask.cpu().numpy(), mask)
    # a stroke over the background after many strokes leaves an all-zero edited mask
    res = ml.apply_stroke(ctx, ml.EditingTool(px=1.0, py=1.0, shape=synth.circle_shape(2), value=9), layer)
    assert res.edited_count == 0 and not bool(res.edited_mask.any())


def test_occlusion_safety_coaxial_quads():                            # SPEC.md:285, 606 acceptance #2
    """Two coaxial quads, many random strokes over the front one: no texel of the occluded quad's
    uv island (right half of the atlas) is ever edited."""
    rng = np.random.default_rng(8)
    mesh = synth.coaxial_quads_mesh()
    A, W = 128, 128
    cam = synth.default_camera(W, W, eye=(0.0, 0.0, 4.0), fovy=40.0, near=0.5, far=10.0)
    surf = ml.build_surface_map(mesh, A, A)
    ctx = ml.StrokeContext(mesh, cam, ml.render_depth(mesh, cam), surf)
    layer = ml.create_layer("L", "uint8", A, A, pool=ml.TexturePool())
    total = 0
    for k in range(200):
        tool = ml.EditingTool(px=float(rng.uniform(20, 108)), py=float(rng.uniform(20, 108)),
                              shape=synth.circle_shape(int(rng.integers(2, 12))), value=1 + k % 200)
        total += ml.apply_stroke(ctx, tool, layer).edited_count
    m = layer.mask.cpu().numpy()
    assert total > 0 and m[:, :A // 2].any()
    assert not m[:, A // 2:].any()


def test_stroke_over_background_and_errors():
    mesh, cam, surf, depth, ctx = _scene()
    layer = ml.create_layer("L", "uint8", 128, 128, pool=ml.TexturePool())
    res = ml.apply_stroke(ctx, ml.EditingTool(px=2.0, py=2.0, shape=synth.circle_shape(2), value=3), layer)
    assert res.edited_count == 0 and layer.valid_texels() == 0
    cam.generation += 1                                              # camera moved, depth not re-rendered
    with pytest.raises(ml.StaleDepth):
        ml.apply_stroke(ctx, ml.EditingTool(px=48.0, py=48.0, shape=synth.circle_shape(8), value=3), layer)
    cam.generation -= 1
    with pytest.raises(ml.TargetMismatch):
        ml.apply_stroke(ctx, ml.EditingTool(px=48.0, py=48.0, shape=synth.circle_shape(8)),
                        ml.create_layer("small", "uint8", 64, 64, pool=ml.TexturePool()))


def test_camera_move_rebuilds_the_stroke_context():                   # SPEC.md:281, 459 (stale MVP)
    """Moving the camera bumps its generation by itself; a stroke with the old depth map raises StaleDepth, and
    once the caller supplies a depth map of the new view the context re-derives its projected triangles, so the
    stroke lands where the oracle puts it for the NEW camera (culled, streamed and one-call paths)."""
    mesh, cam, surf, depth, ctx = _scene()
    A = 128
    tool = ml.EditingTool(px=50.0, py=44.0, shape=synth.circle_shape(10), value=6)
    pool = ml.TexturePool()
    ml.apply_stroke(ctx, tool, ml.create_layer("before", "uint8", A, A, pool=pool))
    g0 = cam.generation
    cam.set_view(synth.look_at((2.0, 1.0, 2.0), (0.0, 0.0, 0.0)))
    assert cam.generation == g0 + 1
    with pytest.raises(ml.StaleDepth):
        ml.apply_stroke(ctx, tool, ml.create_layer("stale", "uint8", A, A, pool=pool))
    ctx.depth = ml.render_depth(mesh, cam)
    data = np.zeros((A, A), np.uint8); mask = np.zeros((A, A), bool); edited = np.zeros((A, A), np.uint8)
    want = _oracle_stroke(mesh, cam, tool, A, data, mask, edited)
    assert want[0] > 0
    outline = ml.build_outline_mask(surf.coverage, thickness=1)
    for mode in ("cull", "stream", "one_call"):
        layer = ml.create_layer(mode, "uint8", A, A, pool=pool)
        if mode == "one_call":
            t0 = ml.EditingTool(px=tool.px, py=tool.py, shape=tool.shape, value=tool.value, padding_radius=1)
            res = ml.stroke(ctx, t0, layer, outline)
            assert (res.edited_count, res.fragments) == want
            assert np.array_equal(res.edited_mask.cpu().numpy(), edited)
        else:
            res = ml.apply_stroke(ctx, tool, layer, cull=(mode == "cull"))
            assert (res.edited_count, res.fragments) == want, mode
            assert np.array_equal(layer.data.cpu().numpy(), data) and np.array_equal(layer.mask.cpu().numpy(), mask)
    # an in-place edit of the matrices (no setter involved) is caught through the MVP bytes in the key
    cam.view[0, 3] += 0.25
    with pytest.raises(ml.StaleDepth):
        ml.apply_stroke(ctx, tool, ml.create_layer("inplace", "uint8", A, A, pool=pool))


def test_stroke_with_padding_equals_oracle():                         # SPEC.md:476, 298, 309; acceptance #4
    mesh, cam, surf, depth, ctx = _scene()
    A = 128
    outline = ml.build_outline_mask(surf.coverage, thickness=1)
    cov = (surf.tri_id >= 0).cpu().numpy()
    ref_outline = kn.outline(cov.astype(np.uint8), 1)
    assert np.array_equal(outline.cpu().numpy(), ref_outline != 0)
    assert not (ref_outline.astype(bool) & cov).any()
    tool = ml.EditingTool(px=48.0, py=48.0, shape=synth.circle_shape(14), value=9, padding_radius=1)
    layer = ml.create_layer("L", "int16", A, A, pool=ml.TexturePool())
    res = ml.stroke(ctx, tool, layer, outline)
    data = np.zeros((A, A), np.int16); mask = np.zeros((A, A), bool); edited = np.zeros((A, A), np.uint8)
    want = _oracle_stroke(mesh, cam, tool, A, data, mask, edited)
    padded = kn.padding(ref_outline, edited, 1, data, mask, 9)
    assert (res.edited_count, res.fragments) == want and res.padded_count == padded > 0
    assert np.array_equal(layer.data.cpu().numpy(), data) and np.array_equal(layer.mask.cpu().numpy(), mask)
    pad_set = mask & ~edited.astype(bool)
    assert pad_set.sum() == padded and not (pad_set & cov).any()                     # disjoint, inside outline


@pytest.mark.parametrize("kind,radius", [("uint8", 1), ("uint8", 4), ("int16", 2), ("uint32", 3)])
def test_culled_stroke_sequence_with_padding_equals_oracle(kind, radius):
    """stroke() = TEA + TPA with footprint culling in BOTH passes, a sequence of strokes on one
    context (the edited mask is only cleared per footprint): planes, edit and padded counts equal
    the oracle after every stroke, and equal the un-culled stroke()."""
    rng = np.random.default_rng(33 + radius)
    mesh = synth.icosphere_mesh(3)
    A, W = 256, 160
    cam = synth.default_camera(W, W)
    surf = ml.build_surface_map(mesh, A, A)
    depth = ml.render_depth(mesh, cam)
    ctx = ml.StrokeContext(mesh, cam, depth, surf)
    ctx_full = ml.StrokeContext(mesh, cam, depth, surf)
    outline = ml.build_outline_mask(surf.coverage, thickness=radius)
    ref_outline = kn.outline((surf.tri_id >= 0).cpu().numpy().astype(np.uint8), radius)
    pool = ml.TexturePool()
    layer = ml.create_layer("L", kind, A, A, pool=pool)
    layer_full = ml.create_layer("F", kind, A, A, pool=pool)
    npk = {"uint8": np.uint8, "int16": np.int16, "uint32": np.uint32}[kind]
    data = np.zeros((A, A), npk); mask = np.zeros((A, A), bool)
    total_padded = 0
    for k in range(8):
        tool = ml.EditingTool(px=float(rng.uniform(30, 130)), py=float(rng.uniform(30, 130)),
                              shape=synth.circle_shape(int(rng.integers(3, 25))), value=k + 1, padding_radius=radius)
        edited = np.zeros((A, A), np.uint8)
        want = _oracle_stroke(mesh, cam, tool, A, data, mask, edited)
        padded = kn.padding(ref_outline, edited, radius, data, mask, k + 1)
        res = ml.stroke(ctx, tool, layer, outline)
        assert ctx.stroke_tiles is not None
        assert (res.edited_count, res.fragments) == want and res.padded_count == padded, k
        got = layer.data.view(_torch_i32()) if kind == "uint32" else layer.data
        assert np.array_equal(got.cpu().numpy().view(npk), data) and np.array_equal(layer.mask.cpu().numpy(), mask)
        res2 = ml.stroke(ctx_full, tool, layer_full, outline, cull=False)
        assert (res2.edited_count, res2.padded_count) == (want[0], padded)
        total_padded += padded
    assert total_padded > 0


def test_row_sharded_strokes_equal_full_plane_oracle():
    """The multi-GPU stroke path on one GPU: three row slabs (heights 100 / 28 / 128, the middle one
    not a multiple of the 8-row tiles) each run the culled TEA + TPA of every stroke, the padding
    halo rows come from the neighbour slabs' edited planes (what sharding.exchange_halo moves);
    stacked slab planes and summed counts == the full-plane oracle after every stroke."""
    import torch
    rng = np.random.default_rng(61)
    mesh = synth.icosphere_mesh(3)
    A, W, radius = 256, 160, 2
    cam = synth.default_camera(W, W)
    depth = ml.render_depth(mesh, cam)
    slabs = [(0, 100), (100, 28), (128, 128)]
    full = ml.build_surface_map(mesh, A, A)
    cov = full.coverage.to(torch.uint8)
    ref_outline = kn.outline(cov.cpu().numpy(), radius)
    pool = ml.TexturePool()
    ctxs, layers, outlines = [], [], []
    for r0, rows in slabs:
        surf = ml.build_surface_map(mesh, A, A, row0=r0, rows=rows)
        ctxs.append(ml.StrokeContext(mesh, cam, depth, surf))
        layers.append(ml.create_layer("s%d" % r0, "uint8", A, rows, pool=pool))
        lo, hi = max(0, r0 - radius), min(A, r0 + rows + radius)
        outlines.append(nat.outline_mask(cov[lo:hi].contiguous(), radius, in_row0=lo, out_row0=r0, out_rows=rows))
    assert np.array_equal(np.concatenate([o.cpu().numpy() for o in outlines]), ref_outline)
    data = np.zeros((A, A), np.uint8); mask = np.zeros((A, A), bool)
    for k in range(6):
        tool = ml.EditingTool(px=float(rng.uniform(40, 120)), py=float(rng.uniform(40, 120)),
                              shape=synth.circle_shape(int(rng.integers(8, 30))), value=k + 1, padding_radius=radius)
        edited = np.zeros((A, A), np.uint8)
        want = _oracle_stroke(mesh, cam, tool, A, data, mask, edited)
        padded = kn.padding(ref_outline, edited, radius, data, mask, k + 1)
        # TEA on every slab first (its edited rows are the neighbours' halos), then the padding passes
        res = [ml.apply_stroke(c, tool, l) for c, l in zip(ctxs, layers)]
        got_padded = 0
        for i, (r0, rows) in enumerate(slabs):
            lo, hi = max(0, r0 - radius), min(A, r0 + rows + radius)
            parts = []
            if lo < r0:
                parts.append(ctxs[i - 1].edited[-(r0 - lo):])
            parts.append(ctxs[i].edited)
            if hi > r0 + rows:
                parts.append(ctxs[i + 1].edited[:hi - (r0 + rows)])
            ext = torch.cat(parts, dim=0)
            got_padded += nat.apply_padding(outlines[i], ext, radius, layers[i].data, layers[i].mask, k + 1,
                                            in_row0=lo, out_row0=r0)
        assert sum(r.edited_count for r in res) == want[0] and sum(r.fragments for r in res) == want[1]
        assert got_padded == padded
        assert np.array_equal(np.concatenate([l.data.cpu().numpy() for l in layers]), data), k
        assert np.array_equal(np.concatenate([l.mask.cpu().numpy() for l in layers]), mask), k
        assert np.array_equal(np.concatenate([c.edited.cpu().numpy() for c in ctxs]), edited), k
    # the public stroke() with an injected halo exchange does the same on one slab
    i, (r0, rows) = 1, slabs[1]
    tool = ml.EditingTool(px=80.0, py=80.0, shape=synth.circle_shape(25), value=9, padding_radius=radius)
    edited = np.zeros((A, A), np.uint8)
    _oracle_stroke(mesh, cam, tool, A, data, mask, edited)
    kn.padding(ref_outline, edited, radius, data, mask, 9)
    for j in (0, 2):
        ml.apply_stroke(ctxs[j], tool, layers[j])

    def halo(plane, row0, height, rad):
        lo, hi = max(0, row0 - rad), min(height, row0 + rows + rad)
        return torch.cat([ctxs[0].edited[-(row0 - lo):], plane, ctxs[2].edited[:hi - (row0 + rows)]], dim=0), lo
    ml.stroke(ctxs[1], tool, layers[1], outlines[1], halo=halo)
    assert np.array_equal(layers[1].data.cpu().numpy(), data[r0:r0 + rows])
    assert np.array_equal(layers[1].mask.cpu().numpy(), mask[r0:r0 + rows])


@pytest.mark.parametrize("radius,slabs", [(1, [(0, 96), (96, 32), (128, 128)]), (2, [(0, 100), (100, 28), (128, 128)]),
                                          (4, [(0, 120), (120, 8), (128, 3), (131, 125)])])
def test_slab_padding_tile_pass_plus_border_rows_equals_full_plane_oracle(radius, slabs):
    """editing.pad_slab (the per-stroke TPA of a row-sharded atlas): footprint-culled tile pass over the
    interior rows + streaming pass over the `radius` border rows with the neighbours' halo rows, on ragged
    slabs (one thinner than the radius window).  Stacked planes and the summed padded count == the
    full-plane oracle after every stroke, strokes centred on the slab borders included."""
    import torch
    from paper_2501_14807_b200 import editing
    rng = np.random.default_rng(67 + radius)
    mesh = synth.icosphere_mesh(3)
    A, W = 256, 160
    cam = synth.default_camera(W, W)
    depth = ml.render_depth(mesh, cam)
    full = ml.build_surface_map(mesh, A, A)
    cov = full.coverage.to(torch.uint8)
    ref_outline = kn.outline(cov.cpu().numpy(), radius)
    pool = ml.TexturePool()
    ctxs, layers, outlines = [], [], []
    for r0, rows in slabs:
        surf = ml.build_surface_map(mesh, A, A, row0=r0, rows=rows)
        ctxs.append(ml.StrokeContext(mesh, cam, depth, surf))
        layers.append(ml.create_layer("p%d" % r0, "uint8", A, rows, pool=pool))
        lo, hi = max(0, r0 - radius), min(A, r0 + rows + radius)
        outlines.append(nat.outline_mask(cov[lo:hi].contiguous(), radius, in_row0=lo, out_row0=r0, out_rows=rows))
    data = np.zeros((A, A), np.uint8); mask = np.zeros((A, A), bool)
    stacked = lambda: torch.cat([c.edited for c in ctxs], 0)             # noqa: E731

    def halo_rows(plane, row0, height, rad):                              # what exchange_halo(parts=True) returns
        allr = stacked()
        rows = plane.shape[0]
        up = allr[max(0, row0 - rad):row0] if row0 > 0 else None
        dn = allr[row0 + rows:min(height, row0 + rows + rad)] if row0 + rows < height else None
        return up, dn
    for k in range(8):
        tool = ml.EditingTool(px=float(rng.uniform(30, 130)), py=float(rng.uniform(30, 130)),
                              shape=synth.circle_shape(int(rng.integers(6, 34))), value=k + 1, padding_radius=radius)
        edited = np.zeros((A, A), np.uint8)
        _oracle_stroke(mesh, cam, tool, A, data, mask, edited)
        padded = kn.padding(ref_outline, edited, radius, data, mask, k + 1)
        for c, l in zip(ctxs, layers):
            ml.apply_stroke(c, tool, l)
        pc = torch.zeros(1, dtype=torch.int64, device="cuda")
        for i, (r0, rows) in enumerate(slabs):
            editing.pad_slab(outlines[i], ctxs[i].edited, radius, layers[i].data, layers[i].mask, k + 1, pc,
                             row0=r0, height=A, tiles=ctxs[i].stroke_tiles, halo=halo_rows)
        assert int(pc.item()) == padded, k
        assert np.array_equal(torch.cat([l.data for l in layers], 0).cpu().numpy(), data), k
        assert np.array_equal(torch.cat([l.mask for l in layers], 0).cpu().numpy(), mask), k
    assert mask.any() and any(c.stroke_tiles is not None for c in ctxs)


def test_stroke_gesture_equals_stroke_loop():
    """ml_stroke_sequence: a drag gesture of 9 strokes (host-side numpy shapes of different sizes,
    different values) in one C call == the same strokes through stroke() one by one == the oracle."""
    rng = np.random.default_rng(71)
    mesh = synth.icosphere_mesh(3)
    A, W = 256, 160
    cam = synth.default_camera(W, W)
    surf = ml.build_surface_map(mesh, A, A)
    depth = ml.render_depth(mesh, cam)
    outline = ml.build_outline_mask(surf.coverage, thickness=1)
    ref_outline = kn.outline((surf.tri_id >= 0).cpu().numpy().astype(np.uint8), 1)
    tools = [ml.EditingTool(px=40.0 + 9.0 * k, py=float(rng.uniform(40, 120)), shape=synth.circle_shape(int(rng.integers(3, 22))),
                            value=k + 1, padding_radius=1) for k in range(9)]
    pool = ml.TexturePool()
    g_layer, l_layer = ml.create_layer("g", "uint8", A, A, pool=pool), ml.create_layer("l", "uint8", A, A, pool=pool)
    g_ctx, l_ctx = ml.StrokeContext(mesh, cam, depth, surf), ml.StrokeContext(mesh, cam, depth, surf)
    ml.stroke(g_ctx, tools[0], g_layer, outline)                      # odd starting parity of the tile buffers
    ml.stroke(l_ctx, tools[0], l_layer, outline)
    got = ml.stroke_gesture(g_ctx, tools, g_layer, outline)
    loop = [ml.stroke(l_ctx, t, l_layer, outline) for t in tools]
    data = np.zeros((A, A), np.uint8); mask = np.zeros((A, A), bool)
    for t in [tools[0]] + tools:
        edited = np.zeros((A, A), np.uint8)
        want = _oracle_stroke(mesh, cam, t, A, data, mask, edited)
        padded = kn.padding(ref_outline, edited, 1, data, mask, t.value)
    assert [(r.edited_count, r.fragments, r.padded_count) for r in got] == [(r.edited_count, r.fragments, r.padded_count) for r in loop]
    assert (got[-1].edited_count, got[-1].fragments, got[-1].padded_count) == (want[0], want[1], padded)
    for layer in (g_layer, l_layer):
        assert np.array_equal(layer.data.cpu().numpy(), data) and np.array_equal(layer.mask.cpu().numpy(), mask)
    assert np.array_equal(g_ctx.edited.cpu().numpy(), edited) and g_ctx.cur == l_ctx.cur
    # a following single stroke continues correctly on both contexts
    extra = ml.EditingTool(px=100.0, py=100.0, shape=synth.square_shape(9), value=77)
    a, b = ml.stroke(g_ctx, extra, g_layer, outline), ml.stroke(l_ctx, extra, l_layer, outline)
    assert a.edited_count == b.edited_count and np.array_equal(g_layer.data.cpu().numpy(), l_layer.data.cpu().numpy())
    assert np.array_equal(g_ctx.edited.cpu().numpy(), l_ctx.edited.cpu().numpy())
    assert ml.stroke_gesture(g_ctx, [], g_layer, outline) == []


def _torch_i32():
    import torch
    return torch.int32


# ------------------------------------------------------------------ display + files (f3)

@pytest.mark.parametrize("kind", ["uint8", "int16", "float32", "float16", "uint32", "int8", "int32"])
def test_resolve_display_matches_oracle(kind):
    import torch
    rng = np.random.default_rng(11)
    h, w = 37, 53
    pal = ml.Palette([0, 0.3, 0.65, 1], rng.random((4, 4)))
    layer = ml.create_layer("L", kind, w, h, palette=pal, limits=(-5.0, 90.0), pool=ml.TexturePool())
    data = (rng.normal(size=(h, w)) * 60).astype(kind)
    mask = rng.random((h, w)) < 0.6
    if kind == "uint32":
        layer.data.view(torch.int32).copy_(torch.from_numpy(data.view(np.int32)))
    else:
        layer.data.copy_(torch.from_numpy(data))
    layer.mask.copy_(torch.from_numpy(mask))
    out = ml.resolve_display(layer).cpu().numpy()
    assert out.shape == (h, w, 4)
    assert np.array_equal(out, kn.resolve_display(data, mask.view(np.uint8), -5.0, 90.0, pal.positions, pal.colours))
    assert (out[~mask] == 0).all()


def test_display_known_answers_and_pack():
    import torch
    layer = ml.create_layer("L", "float32", 8, 8, limits=(0.0, 10.0), pool=ml.TexturePool())
    assert not bool(ml.resolve_display(layer).any())                                 # all-false mask
    layer.data[3, 3] = 5.0
    layer.mask[3, 3] = True
    out = ml.resolve_display(layer).cpu().numpy()
    assert out[3, 3].tolist() == [128, 128, 128, 255] and (out.reshape(-1, 4).any(axis=1).sum() == 1)
    for n in (1, 7, 8, 9, 1000, 4099):
        m = (np.random.default_rng(n).random(n) < 0.4).astype(np.uint8) * 3
        bits = nat.pack_mask(_dev(m))
        assert np.array_equal(bits.cpu().numpy(), np.packbits(m != 0))
        back = torch.empty(n, dtype=torch.uint8, device="cuda")
        assert np.array_equal(nat.unpack_mask(bits, n, back).cpu().numpy(), (m != 0).astype(np.uint8))


@pytest.mark.parametrize("seed", range(10))
def test_save_load_layer_bit_identical(seed):                         # SPEC.md:207, 613 acceptance #9
    import torch
    rng = np.random.default_rng(600 + seed)
    kind = ["int8", "int16", "int32", "uint8", "float16", "float32", "uint32"][seed % 7]
    w, h = int(rng.integers(1, 90)), int(rng.integers(1, 90))
    pal = ml.Palette(np.array([0, 0.5, 1], np.float32), rng.random((3, 4)).astype(np.float32))
    layer = ml.create_layer("orig", kind, w, h, palette=pal, limits=(-1.0, 7.5), pool=ml.TexturePool(),
                            table="records" if kind == "uint32" else None)
    data = (rng.normal(size=(h, w)) * 50).astype(kind)
    mask = rng.random((h, w)) < 0.5
    (layer.data.view(torch.int32) if kind == "uint32" else layer.data).copy_(
        torch.from_numpy(data.view(np.int32) if kind == "uint32" else data))
    layer.mask.copy_(torch.from_numpy(mask))
    blob = ml.save_layer(layer)
    back = ml.load_layer(blob, name="copy", pool=ml.TexturePool())
    got = back.data.view(torch.int32).cpu().numpy().view(np.uint32) if kind == "uint32" else back.data.cpu().numpy()
    assert np.array_equal(got.view(np.uint8), data.view(np.uint8)) and np.array_equal(back.mask.cpu().numpy(), mask)
    assert back.kind == kind and back.limits == (-1.0, 7.5) and back.table == layer.table
    assert np.array_equal(back.palette.colours, pal.colours) and ml.save_layer(back) == blob
    with pytest.raises(ml.ChecksumMismatch):
        ml.load_layer(blob[:-1] + bytes([blob[-1] ^ 1]))


# ------------------------------------------------------------------ engine-level algebra / area API

def test_layer_algebra_and_area_api():
    mesh, cam, surf, depth, ctx = _scene()
    pool = ml.TexturePool()
    a, b, c = (ml.create_layer(n, "uint8", 128, 128, pool=pool) for n in "abc")
    ml.select_sphere(surf, a, (0.0, 0.0, 1.0), 0.5, 3)
    ml.select_sphere(surf, b, (0.4, 0.0, 0.9), 0.5, 5)
    na, nb = a.valid_texels(), b.valid_texels()
    u = ml.layer_union(a, b, out=c)
    nu = u.valid_texels()
    i = ml.layer_intersection(a, b, out=ml.create_layer("i", "uint8", 128, 128, pool=pool))
    d = ml.layer_difference(a, b, out=ml.create_layer("d", "uint8", 128, 128, pool=pool))
    assert nu == na + nb - i.valid_texels() and d.valid_texels() == na - i.valid_texels()
    areas, counts = ml.layers_area([a, b, u, i, d], surf)
    assert counts.tolist() == [na, nb, nu, i.valid_texels(), d.valid_texels()]
    assert abs(areas[2] - (areas[0] + areas[1] - areas[3])) < 1e-9 * areas[2]        # inclusion-exclusion
    assert abs(ml.layer_area(d, surf) - areas[4]) < 1e-12
    chain = ml.layer_chain([a, b, i], ["union", "difference"], ml.create_layer("x", "uint8", 128, 128, pool=pool))
    assert chain.valid_texels() == nu - i.valid_texels()
    lab_area, lab_count = ml.label_area(u, surf)
    assert lab_count[3] == na and lab_count[5] == nu - na and abs(lab_area.sum() - areas[2]) < 1e-9 * areas[2]
    cnt, s, mn, mx = ml.layer_stats(u)
    assert (cnt, mn, mx) == (nu, 3.0, 5.0) and s == 3.0 * na + 5.0 * (nu - na)
    with pytest.raises(ml.TargetMismatch):
        ml.layer_union(a, ml.create_layer("small", "uint8", 64, 64, pool=pool))


def test_edit_result_duration_and_gesture_masks():
    mesh, cam, surf, depth, ctx = _scene()
    A = 128
    outline = ml.build_outline_mask(surf.coverage, thickness=1)
    layer = ml.create_layer("L", "uint8", A, A, pool=ml.TexturePool())
    tool = ml.EditingTool(px=48.0, py=48.0, shape=synth.circle_shape(10), value=4)
    assert ml.stroke(ctx, tool, layer, outline).duration_ms is None           # nobody asked: no events on the stroke path
    r = ml.stroke(ctx, tool, layer, outline, timed=True)
    assert r.duration_ms is not None and 0.0 < r.duration_ms < 1000.0
    tools = [ml.EditingTool(px=30.0 + 9 * k, py=50.0, shape=synth.circle_shape(6), value=5 + k) for k in range(4)]
    res = ml.stroke_gesture(ctx, tools, layer, outline)
    assert [x.edited_mask is None for x in res] == [True, True, True, False]   # one EditedAreaMask per context
    assert int(res[-1].edited_mask.sum().item()) == res[-1].edited_count > 0


def test_rasterize_discarded_triangle_does_not_hide_a_kept_one():
    """A texel covered by a kept triangle and by a LATER discarded triangle holds the kept triangle's value,
    and the written count includes it."""
    pool = ml.TexturePool()
    big = np.array([[[0.0, 0.0], [8.0, 0.0], [0.0, 8.0]]])                     # covers the lower-left half
    later = np.array([[[0.0, 0.0], [4.0, 0.0], [0.0, 4.0]]])                   # inside it, submitted later
    tri = np.concatenate([big, later])
    a = pool.acquire(8, 8, "uint8")
    n_all = ml.rasterize(tri, [a], [np.array([3, 9])])
    got_all = a.tensor.cpu().numpy().copy()
    assert (got_all == 9).sum() > 0 and (got_all == 3).sum() > 0               # last submission wins on the overlap
    b = pool.acquire(8, 8, "uint8")
    n_kept = ml.rasterize(tri, [b], [np.array([3, 9])], keep=[True, False])
    c = pool.acquire(8, 8, "uint8")
    n_big = ml.rasterize(big, [c], [3])
    assert n_kept == n_big == n_all
    assert np.array_equal(b.tensor.cpu().numpy(), c.tensor.cpu().numpy())     # the discarded triangle left no hole


def test_rasterize_known_answers():
    """rule "always keep, write 7" fills exactly the covered centres; "always
    discard" writes nothing; two overlapping triangles writing 1 then 2 leave 2 on the overlap; targets
    of different dimensions raise TargetMismatch."""
    import torch
    pool = ml.TexturePool()
    tri = np.array([[[1.0, 1.0], [3.2, 1.0], [1.0, 3.2]]])                         # covers centres (1,1), (2,1), (1,2)
    a = pool.acquire(6, 6, "uint8")
    assert ml.rasterize(tri, [a], [7]) == 3
    got = a.tensor.cpu().numpy()
    want = np.zeros((6, 6), np.uint8); want[1, 1] = want[1, 2] = want[2, 1] = 7     # [row=y, col=x]
    assert np.array_equal(got, want)
    ref = np.zeros((6, 6), np.uint8)
    assert kn.coverage_fill(tri, 6, 6, ref) == 3 and np.array_equal(ref * 7, want)
    b = pool.acquire(6, 6, "int16")
    assert ml.rasterize(tri, [b], [5], keep=[False]) == 0 and not bool(b.tensor.any())          # always discard
    two = np.array([[[0.0, 0.0], [5.0, 0.0], [0.0, 5.0]], [[1.0, 1.0], [6.0, 1.0], [1.0, 6.0]]])
    c, d = pool.acquire(6, 6, "uint8"), pool.acquire(6, 6, "float32")
    n = ml.rasterize(two, [c, d], [np.array([1, 2]), np.array([0.5, 0.25])])
    r1, r2 = np.zeros((6, 6), np.uint8), np.zeros((6, 6), np.uint8)
    kn.coverage_fill(two[:1], 6, 6, r1); kn.coverage_fill(two[1:], 6, 6, r2)
    exp = np.where(r2 != 0, 2, r1).astype(np.uint8)                                # submission order: 2 wins on overlap
    assert n == int((exp != 0).sum()) and np.array_equal(c.tensor.cpu().numpy(), exp)
    assert np.array_equal(d.tensor.cpu().numpy(), np.where(exp == 2, 0.25, np.where(exp == 1, 0.5, 0.0)).astype(np.float32))
    with pytest.raises(ml.TargetMismatch):
        ml.rasterize(tri, [a, pool.acquire(8, 6, "uint8")], [1, 1])
    assert ml.rasterize(np.zeros((0, 3, 2)), [a], [1]) == 0


def test_non_square_atlas_and_window_whole_pipeline():
    """Atlas 384 x 200 (wider than tall, height not a multiple of the 4- / 8-row tiles) and a 160 x 96
    window: surface map, culled strokes with padding (one-call stroke), culled sphere brush, culled
    height threshold and areas all == oracle."""
    import torch
    rng = np.random.default_rng(91)
    mesh = synth.icosphere_mesh(3)
    AW, AH, WW, WH = 384, 200, 160, 96
    cam = synth.default_camera(WW, WH)
    surf = ml.build_surface_map(mesh, AW, AH)
    txy = mesh.tri_uv_texels(AW, AH)
    ref = kn.surface_map(txy, mesh.tri_pos(), mesh.tri_nrm(), AW, AH)
    assert np.array_equal(surf.tri_id.cpu().numpy(), ref["tri_id"]) and surf.tiles is not None
    assert np.array_equal(surf.pos.cpu().numpy().view(np.uint32), ref["pos"].view(np.uint32))
    depth = ml.render_depth(mesh, cam)
    xy, zn = window_triangles(mesh, cam)
    d_ref = np.ones((WH, WW), np.float32)
    kn.raster_depth(xy, zn, d_ref)
    assert np.array_equal(depth.plane.cpu().numpy().view(np.uint32), d_ref.view(np.uint32))
    ctx = ml.StrokeContext(mesh, cam, depth, surf)
    outline = ml.build_outline_mask(surf.coverage, thickness=1)
    ref_outline = kn.outline((ref["tri_id"] >= 0).astype(np.uint8), 1)
    assert np.array_equal(outline.cpu().numpy(), ref_outline != 0)
    pool = ml.TexturePool()
    layer = ml.create_layer("L", "uint8", AW, AH, pool=pool)
    data = np.zeros((AH, AW), np.uint8); mask = np.zeros((AH, AW), bool)
    clip = cam.clip_coords(mesh.vertices)[mesh.triangles]
    for k in range(5):
        tool = ml.EditingTool(px=float(rng.uniform(30, 130)), py=float(rng.uniform(20, 76)),
                              shape=synth.circle_shape(int(rng.integers(4, 20))), value=k + 1)
        sfx, sfy, bx, by = ml.compute_tool_projection(cam, tool).kernel_factors
        edited = np.zeros((AH, AW), np.uint8)
        want = kn.raster_tea(txy, clip, float(WW), float(WH), d_ref, 1e-4, sfx, sfy, bx, by, tool.shape, data, mask, edited, k + 1)
        padded = kn.padding(ref_outline, edited, 1, data, mask, k + 1)
        res = ml.stroke(ctx, tool, layer, outline)
        assert (res.edited_count, res.fragments, res.padded_count) == (want[0], want[1], padded), k
        assert np.array_equal(layer.data.cpu().numpy(), data) and np.array_equal(layer.mask.cpu().numpy(), mask)
    ed = torch.zeros((AH, AW), dtype=torch.uint8, device="cuda")
    e_ref = np.zeros((AH, AW), np.uint8)
    n = kn.select_sphere(ref["pos"], (0.2, 0.1, 0.95), 0.35, data, mask, e_ref, 9)
    assert ml.select_sphere(surf, layer, (0.2, 0.1, 0.95), 0.35, 9, edited=ed).edited_count == n > 0
    tiles = nat.attr_tiles(surf.pos[2])
    n = kn.select_threshold(np.ascontiguousarray(ref["pos"][2]), None, -0.1, 0.2, data, mask, e_ref, 11)
    assert ml.select_threshold(surf.pos[2], None, -0.1, 0.2, layer, 11, edited=ed, tiles=tiles).edited_count == n > 0
    assert np.array_equal(layer.data.cpu().numpy(), data) and np.array_equal(layer.mask.cpu().numpy(), mask)
    assert np.array_equal(ed.cpu().numpy(), e_ref)
    a_ref = kn.layer_area(ref["area"], mask.astype(np.uint8))[0]
    assert abs(ml.layer_area(layer, surf) - a_ref) <= 1e-9 * a_ref
