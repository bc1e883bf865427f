"""Parity at BASELINE.json's full sizes (16384^2 atlas, ~1M triangles) through size-independent
properties -- the oracle cannot run these sizes in seconds, so the checks are algebraic
identities, idempotence, slab-vs-full checksums and a sampled comparison against the oracle on
a thin row slab."""
import numpy as np
import pytest

import paper_2501_14807_b200 as ml
from oracle import kn
from paper_2501_14807_b200 import _native as nat
from paper_2501_14807_b200 import synth

pytestmark = pytest.mark.gpu

A = 16384


def _checksum(t):
    """Order-independent 64-bit checksum of a plane (sum of (index+1) * (value+1) mod 2^63)."""
    import torch
    v = t.reshape(-1).to(torch.int64)
    idx = torch.arange(1, v.numel() + 1, device=t.device, dtype=torch.int64)
    return int(((v + 1) * idx).sum().item())


@pytest.fixture(scope="module")
def big():
    mesh = synth.heightfield_mesh(707, margin=0.01)                 # 999,698 triangles (C2 mesh)
    surf = ml.build_surface_map(mesh, A, A)
    cam = synth.default_camera(1024, 1024, eye=(0.5, 0.5, 1.6), target=(0.5, 0.5, 0.0), fovy=40.0, near=0.2, far=5.0)
    depth = ml.render_depth(mesh, cam)
    ctx = ml.StrokeContext(mesh, cam, depth, surf)
    pool = ml.TexturePool(budget_texels=40 * A * A)
    return mesh, surf, cam, ctx, pool


def test_surface_map_full_size_properties(big):
    mesh, surf, cam, ctx, pool = big
    assert surf.overlap == 0 and surf.fragments == surf.covered
    assert int((surf.tri_id >= 0).sum().item()) == surf.covered
    # every covered texel has a finite position, uncovered ones NaN; area integrates to the mesh area
    import torch
    cov = surf.tri_id >= 0
    assert bool(torch.isfinite(surf.pos[:, cov]).all()) and bool(torch.isnan(surf.pos[0][~cov]).all())
    sums, counts = nat.layer_area(surf.area, [cov.to(torch.uint8)])
    assert counts[0] == surf.covered
    assert abs(sums[0] - ml.mesh_surface_area(mesh)) / ml.mesh_surface_area(mesh) < 2e-3
    # a thin slab of the full-size map equals the oracle bit for bit (sampled parity at full size)
    r0, r1 = 8000, 8016
    ref = kn.surface_map(mesh.tri_uv_texels(A, A), mesh.tri_pos(), mesh.tri_nrm(), A, A, rows=(r0, r1))
    assert np.array_equal(surf.tri_id[r0:r1].cpu().numpy(), ref["tri_id"])
    assert np.array_equal(surf.pos[:, r0:r1].cpu().numpy().view(np.uint32), ref["pos"].view(np.uint32))
    assert np.array_equal(surf.area[r0:r1].cpu().numpy().view(np.uint32), ref["area"].view(np.uint32))


def test_slab_equals_full_at_full_size(big):
    """Row sharding: a 4096-row slab built on its own has the same checksums as the same rows of
    the full map (what an 4-GPU row-sharded run would hold)."""
    mesh, surf, cam, ctx, pool = big
    r0, rows = 4096, 4096
    part = ml.build_surface_map(mesh, A, A, row0=r0, rows=rows)
    assert _checksum(part.tri_id) == _checksum(surf.tri_id[r0:r0 + rows])
    import torch
    assert _checksum(part.pos.view(torch.int32)) == _checksum(surf.pos[:, r0:r0 + rows].contiguous().view(torch.int32))
    assert _checksum(part.area.view(torch.int32)) == _checksum(surf.area[r0:r0 + rows].contiguous().view(torch.int32))


def test_strokes_idempotent_and_algebra_identities(big):
    mesh, surf, cam, ctx, pool = big
    import torch
    a = ml.create_layer("a", "uint8", A, A, pool=pool)
    b = ml.create_layer("b", "uint8", A, A, pool=pool)
    tool = ml.EditingTool(px=500.0, py=520.0, shape=synth.circle_shape(70), value=7)
    first = ml.apply_stroke(ctx, tool, a)
    n1, frags = first.edited_count, first.fragments
    assert n1 > 0 and frags == surf.covered                         # SPEC.md:310 every covered texel once
    snap = a.data.clone()
    again = ml.apply_stroke(ctx, tool, a)                           # idempotence
    assert again.edited_count == n1 and bool((a.data == snap).all()) and a.valid_texels() == n1
    # the direct per-triangle kernel agrees with the cached per-texel kernel at full size
    direct = ml.create_layer("direct", "uint8", A, A, pool=pool)
    rd = ml.apply_stroke(ctx, tool, direct, force_direct=True)
    assert (rd.edited_count, rd.fragments) == (n1, frags)
    assert _checksum(direct.data) == _checksum(a.data) and _checksum(direct.mask.view(torch.uint8)) == _checksum(a.mask.view(torch.uint8))
    # sphere strokes + algebra identities
    strokes, labels = synth.sphere_strokes(mesh, 6, seed=5, rmin_frac=0.03, rmax_frac=0.1)
    for k in range(3):
        ml.select_sphere(surf, a, strokes[k, :3], strokes[k, 3], int(labels[k]))
        ml.select_sphere(surf, b, strokes[3 + k, :3], strokes[3 + k, 3], int(labels[3 + k]))
    u = ml.layer_union(a, b, out=ml.create_layer("u", "uint8", A, A, pool=pool))
    i = ml.layer_intersection(a, b, out=ml.create_layer("i", "uint8", A, A, pool=pool))
    d = ml.layer_difference(a, b, out=ml.create_layer("d", "uint8", A, A, pool=pool))
    areas, counts = ml.layers_area([a, b, u, i, d], surf)
    assert counts[2] == counts[0] + counts[1] - counts[3] and counts[4] == counts[0] - counts[3]
    assert abs(areas[2] - (areas[0] + areas[1] - areas[3])) <= 1e-9 * areas[2]
    # (A \ B) u (A n B) == A, planes bit-identical
    back = ml.layer_union(d, i, out=ml.create_layer("back", "uint8", A, A, pool=pool))
    assert _checksum(back.mask.view(torch.uint8)) == _checksum(a.mask.view(torch.uint8))
    assert _checksum(back.data) == _checksum(a.data)
    # fused chain == step-by-step
    c1 = ml.layer_chain([a, b, i], ["union", "difference"], ml.create_layer("c1", "uint8", A, A, pool=pool))
    c2 = ml.layer_difference(u, i, out=ml.create_layer("c2", "uint8", A, A, pool=pool))
    assert _checksum(c1.data) == _checksum(c2.data) and c1.valid_texels() == c2.valid_texels()
    # label areas partition the union's area
    la, lc = ml.label_area(u, surf)
    assert lc.sum() == counts[2] and abs(la.sum() - areas[2]) <= 1e-9 * areas[2]


def test_culled_brushes_equal_streamed_at_full_size(big):
    """16384^2: the footprint-culled sphere brush (single and batched) gives the planes and counts of
    the whole-map streaming kernels."""
    mesh, surf, cam, ctx, pool = big
    import torch
    assert surf.tiles is not None
    strokes, labels = synth.sphere_strokes(mesh, 6, seed=13, rmin_frac=0.002, rmax_frac=0.08)
    a = ml.create_layer("cull", "uint8", A, A, pool=pool)
    b = ml.create_layer("full", "uint8", A, A, pool=pool)
    ea = torch.zeros((A, A), dtype=torch.uint8, device="cuda")
    eb = torch.zeros((A, A), dtype=torch.uint8, device="cuda")
    for k in range(6):
        ra = ml.select_sphere(surf, a, strokes[k, :3], strokes[k, 3], int(labels[k]), edited=ea)
        rb = ml.select_sphere(surf, b, strokes[k, :3], strokes[k, 3], int(labels[k]), edited=eb, cull=False)
        assert ra.edited_count == rb.edited_count
    assert _checksum(a.data) == _checksum(b.data) and _checksum(ea) == _checksum(eb)
    assert _checksum(a.mask.view(torch.uint8)) == _checksum(b.mask.view(torch.uint8))
    a2 = ml.create_layer("cull2", "uint8", A, A, pool=pool)
    b2 = ml.create_layer("full2", "uint8", A, A, pool=pool)
    ea.zero_(); eb.zero_()
    lo = np.zeros(6, np.int64)
    ba = nat.StrokeBatch([a2.data], [a2.mask], [ea], "cuda").upload(strokes, lo, labels)
    bb = nat.StrokeBatch([b2.data], [b2.mask], [eb], "cuda").upload(strokes, lo, labels)
    ml.select_sphere_batch(surf, ba)
    ml.select_sphere_batch(surf, bb, cull=False)
    assert int(ba.counts[0]) == int(bb.counts[0]) > 0
    assert _checksum(a2.data) == _checksum(b2.data) and _checksum(ea) == _checksum(eb)
    assert _checksum(a2.data) == _checksum(a.data)               # batch == sequential
    for l in (a, b, a2, b2):
        l.release()


def test_culled_threshold_equals_streamed_at_full_size(big):
    """16384^2: threshold selection on the height plane with tile ranges == the streaming kernel."""
    mesh, surf, cam, ctx, pool = big
    import torch
    attr = surf.pos[2]
    tiles = nat.attr_tiles(attr)
    z = mesh.vertices[:, 2]
    a = ml.create_layer("thr_cull", "uint8", A, A, pool=pool)
    b = ml.create_layer("thr_full", "uint8", A, A, pool=pool)
    ea = torch.zeros((A, A), dtype=torch.uint8, device="cuda")
    eb = torch.zeros((A, A), dtype=torch.uint8, device="cuda")
    for k, (p0, p1) in enumerate(((40, 60), (0, 3), (99.5, 100), (10, 90))):
        lo, hi = float(np.percentile(z, p0)), float(np.percentile(z, p1))
        ra = ml.select_threshold(attr, None, lo, hi, a, k + 1, edited=ea, tiles=tiles)
        rb = ml.select_threshold(attr, None, lo, hi, b, k + 1, edited=eb)
        assert ra.edited_count == rb.edited_count
        assert _checksum(a.data) == _checksum(b.data) and _checksum(ea) == _checksum(eb)
    assert _checksum(a.mask.view(torch.uint8)) == _checksum(b.mask.view(torch.uint8)) and a.valid_texels() > 0
    a.release(); b.release()


def test_batched_strokes_equal_sequential_at_full_size(big):
    mesh, surf, cam, ctx, pool = big
    import torch
    K, L = 48, 4
    strokes, labels = synth.sphere_strokes(mesh, K, seed=9, rmin_frac=0.01, rmax_frac=0.06)
    layer_of = np.arange(K) % L
    seq = [ml.create_layer("s%d" % l, "uint8", A, A, pool=pool) for l in range(L)]
    seq_ed = [torch.zeros((A, A), dtype=torch.uint8, device="cuda") for _ in range(L)]
    want = np.zeros(L, np.int64)
    for k in range(K):
        want[layer_of[k]] += ml.select_sphere(surf, seq[layer_of[k]], strokes[k, :3], strokes[k, 3], int(labels[k]),
                                              edited=seq_ed[layer_of[k]]).edited_count
    bat = [ml.create_layer("b%d" % l, "uint8", A, A, pool=pool) for l in range(L)]
    bat_ed = [torch.zeros((A, A), dtype=torch.uint8, device="cuda") for _ in range(L)]
    batch = nat.StrokeBatch([l.data for l in bat], [l.mask for l in bat], bat_ed, "cuda").upload(strokes, layer_of, labels)
    ml.select_sphere_batch(surf, batch)
    assert np.array_equal(batch.counts.cpu().numpy(), want)
    for l in range(L):
        assert _checksum(bat[l].data) == _checksum(seq[l].data)
        assert _checksum(bat[l].mask.view(torch.uint8)) == _checksum(seq[l].mask.view(torch.uint8))


def test_row_sharded_stroke_with_padding_equals_whole_plane_at_full_size(big):
    """Two 8192-row slabs of the 16384^2 atlas (what a 2-GPU run holds) each run the culled TEA of a stroke
    that straddles the slab border, then editing.pad_slab with the neighbour's halo row; stacked planes and
    summed counts equal the whole-plane stroke() (ml_stroke: TEA + tile-culled TPA in one call)."""
    import torch
    from paper_2501_14807_b200 import editing
    mesh, surf, cam, ctx, pool = big
    outline = ml.build_outline_mask(surf.coverage, thickness=1)
    # a tool whose footprint crosses atlas row 8192: project the surface point at uv = (0.5, 0.5) into the window
    tool = ml.EditingTool(px=512.0, py=512.0, shape=synth.circle_shape(70), value=11, padding_radius=1)
    whole = ml.create_layer("whole", "uint8", A, A, pool=pool)
    res = ml.stroke(ctx, tool, whole, outline)
    want = (res.edited_count, res.padded_count)
    ed = ctx.edited.clone()
    assert bool(ed[:A // 2].any()) and bool(ed[A // 2:].any())            # the stroke really straddles the border
    assert want[1] >= 0
    halves, layers = [], []
    for r0 in (0, A // 2):
        s = ml.build_surface_map(mesh, A, A, row0=r0, rows=A // 2)
        c = ml.StrokeContext(mesh, cam, ctx.depth, s)
        l = ml.create_layer("half%d" % r0, "uint8", A, A // 2, pool=pool)
        halves.append(c); layers.append(l)
    got_e = sum(ml.apply_stroke(c, tool, l).edited_count for c, l in zip(halves, layers))
    assert torch.equal(torch.cat([c.edited for c in halves], 0), ed)
    pc = torch.zeros(1, dtype=torch.int64, device="cuda")

    def halo(plane, row0, height, rad):
        other = halves[1].edited if row0 == 0 else halves[0].edited
        return (None, other[:rad]) if row0 == 0 else (other[-rad:], None)
    for i, r0 in enumerate((0, A // 2)):
        editing.pad_slab(outline[r0:r0 + A // 2].view(torch.uint8), halves[i].edited, 1, layers[i].data, layers[i].mask,
                         tool.value, pc, row0=r0, height=A, tiles=halves[i].stroke_tiles, halo=halo)
    assert (got_e, int(pc.item())) == want
    assert torch.equal(torch.cat([l.data for l in layers], 0), whole.data)
    assert torch.equal(torch.cat([l.mask for l in layers], 0), whole.mask)
    for l in layers + [whole]:
        l.release() if hasattr(l, "release") else None
