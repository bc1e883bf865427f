"""BASELINE.json's five configurations as parity cases (SURVEY.md 8(d) workload definitions).

C1 and C2 are small enough for the oracle (oracle/kn_port.c) to produce the full expected planes;
C4 and C5 run at their full sizes through size-independent properties (batched == sequential,
culled == streamed, slab == full map, area identities).  C3 (16384^2 x 8 layers: algebra chain +
threshold) lives in test_gpu_fullsize.py."""
import numpy as np
import pytest

import paper_2501_14807_b200 as ml
from oracle import kn
from paper_2501_14807_b200 import _native as nat
from paper_2501_14807_b200 import sharding, synth
from paper_2501_14807_b200.mesh_core import window_triangles

pytestmark = pytest.mark.gpu


def _checksum(t):
    import torch
    v = t.reshape(-1).to(torch.int64)
    idx = torch.arange(1, v.numel() + 1, device=t.device, dtype=torch.int64)
    return int(((v + 1) * idx).sum().item())


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


# ------------------------------------------------------------------ C1

def test_config1_icosphere_1024_single_strokes_equal_oracle():
    """C1: icosphere level 5 (20,480 triangles), 1024^2 chart-grid atlas, camera at z=+3 / 45 deg /
    512^2 window; one TEA stroke (r = 40 px at the window centre, eps 1e-4, value 7) and one
    sphere-brush stroke (centre (0,0,1), radius 0.25): surface map, planes and counts == oracle."""
    A, W = 1024, 512
    mesh = synth.icosphere_mesh(5)
    assert mesh.num_triangles == 20480
    cam = synth.default_camera(W, W)
    surf = ml.build_surface_map(mesh, A, A)
    ref = kn.surface_map(mesh.tri_uv_texels(A, A), mesh.tri_pos(), mesh.tri_nrm(), A, A)
    assert surf.covered == ref["covered"] and surf.overlap == 0
    assert np.array_equal(surf.tri_id.cpu().numpy(), ref["tri_id"])
    for k, t in (("pos", surf.pos), ("nrm", surf.nrm), ("area", surf.area)):
        assert np.array_equal(_bits(t.cpu().numpy()), _bits(ref[k])), k                  # bit-exact (north star: 1e-5)
    # areas: per-texel areas sum to the mesh area (SPEC.md:78-80 anchor, coarse because of the gutters)
    depth = ml.render_depth(mesh, cam)
    xy, zn = window_triangles(mesh, cam)
    d_ref = np.ones((W, W), np.float32)
    kn.raster_depth(xy, zn, d_ref)
    assert np.array_equal(_bits(depth.plane.cpu().numpy()), _bits(d_ref))
    ctx = ml.StrokeContext(mesh, cam, depth, surf)
    pool = ml.TexturePool()
    tool = ml.EditingTool(px=256.0, py=256.0, shape=synth.circle_shape(40), value=7)
    layer = ml.create_layer("tea", "uint8", A, A, pool=pool)
    res = ml.apply_stroke(ctx, tool, layer)
    sfx, sfy, bx, by = ml.compute_tool_projection(cam, tool).kernel_factors
    data = np.zeros((A, A), np.uint8); mask = np.zeros((A, A), bool); edited = np.zeros((A, A), np.uint8)
    want = kn.raster_tea(mesh.tri_uv_texels(A, A), cam.clip_coords(mesh.vertices)[mesh.triangles], float(W), float(W),
                         d_ref, 1e-4, sfx, sfy, bx, by, tool.shape, data, mask, edited, 7)
    assert (res.edited_count, res.fragments) == want and want[0] > 1000
    assert np.array_equal(layer.data.cpu().numpy(), data) and np.array_equal(layer.mask.cpu().numpy(), mask)
    assert np.array_equal(res.edited_mask.cpu().numpy(), edited)
    sl = ml.create_layer("sphere", "uint8", A, A, pool=pool)
    got = ml.select_sphere(surf, sl, (0.0, 0.0, 1.0), 0.25, 3)
    sd = np.zeros((A, A), np.uint8); sm = np.zeros((A, A), bool); se = np.zeros((A, A), np.uint8)
    n = kn.select_sphere(ref["pos"], (0.0, 0.0, 1.0), 0.25, sd, sm, se, 3)
    assert got.edited_count == n > 0
    assert np.array_equal(sl.data.cpu().numpy(), sd) and np.array_equal(sl.mask.cpu().numpy(), sm)
    a_gpu = ml.layer_area(sl, surf)
    a_ref = kn.layer_area(ref["area"], sm.astype(np.uint8))[0]
    assert abs(a_gpu - a_ref) <= 1e-6 * a_ref                                            # north star tolerance


# ------------------------------------------------------------------ C2

@pytest.fixture(scope="module")
def c2():
    A = 4096
    mesh = synth.heightfield_mesh(707)                                # 999,698 triangles
    surf = ml.build_surface_map(mesh, A, A)
    strokes, labels = synth.sphere_strokes(mesh, 1000)                # seeded, radii 0.5%..5% of the diagonal
    return A, mesh, surf, strokes, labels


def test_config2_surface_map_and_first_strokes_equal_oracle(c2):
    """C2: ~1M-triangle heightfield, 4096^2 atlas.  The surface map and the first 48 of the 1000
    strokes (sequential and batched, culled and streamed) + the per-label area == oracle."""
    import torch
    A, mesh, surf, strokes, labels = c2
    assert mesh.num_triangles == 999698
    ref = kn.surface_map(mesh.tri_uv_texels(A, A), mesh.tri_pos(), mesh.tri_nrm(), A, A)
    assert surf.covered == ref["covered"] and surf.overlap == 0
    assert np.array_equal(surf.tri_id.cpu().numpy(), ref["tri_id"])
    for k, t in (("pos", surf.pos), ("nrm", surf.nrm), ("area", surf.area)):
        assert np.array_equal(_bits(t.cpu().numpy()), _bits(ref[k])), k
    K = 48
    rd = np.zeros((A, A), np.uint8); rm = np.zeros((A, A), bool); re = np.zeros((A, A), np.uint8)
    want = 0
    for k in range(K):
        want += kn.select_sphere(ref["pos"], strokes[k, :3], strokes[k, 3], rd, rm, re, labels[k], threads=kn.max_threads())
    pool = ml.TexturePool(budget_texels=64 * A * A)
    for mode in ("sequential-culled", "sequential-streamed", "batch-culled", "batch-streamed"):
        layer = ml.create_layer(mode, "uint8", A, A, pool=pool)
        ed = torch.zeros((A, A), dtype=torch.uint8, device="cuda")
        cull = mode.endswith("culled")
        if mode.startswith("sequential"):
            got = sum(ml.select_sphere(surf, layer, strokes[k, :3], strokes[k, 3], int(labels[k]), edited=ed,
                                       cull=cull).edited_count for k in range(K))
        else:
            batch = nat.StrokeBatch([layer.data], [layer.mask], [ed], "cuda").upload(strokes[:K], np.zeros(K, np.int64), labels[:K])
            got = int(ml.select_sphere_batch(surf, batch, cull=cull)[0])
        assert got == want, mode
        assert np.array_equal(layer.data.cpu().numpy(), rd), mode
        assert np.array_equal(layer.mask.cpu().numpy(), rm) and np.array_equal(ed.cpu().numpy(), re), mode
    la, lc = ml.label_area(layer, surf)
    ra, rc = kn.label_area(ref["area"], rd, rm.astype(np.uint8))
    assert np.array_equal(lc, rc) and np.allclose(la, ra, rtol=1e-9, atol=0.0)


def test_config2_thousand_strokes_and_area(c2):
    """All 1000 strokes: one batched culled pass == 1000 sequential culled strokes == one batched
    streamed pass; label areas partition the layer's area (1e-6 relative, north star)."""
    import torch
    A, mesh, surf, strokes, labels = c2
    K = 1000
    pool = ml.TexturePool(budget_texels=64 * A * A)
    planes = {}
    for mode in ("sequential", "batch-culled", "batch-streamed"):
        layer = ml.create_layer(mode, "uint8", A, A, pool=pool)
        ed = torch.zeros((A, A), dtype=torch.uint8, device="cuda")
        if mode == "sequential":
            counts = torch.zeros(1, dtype=torch.int64, device="cuda")
            for k in range(K):
                nat.select_sphere(surf.pos, strokes[k, :3], strokes[k, 3], layer.data, layer.mask, ed, int(labels[k]),
                                  counts=counts, tiles=surf.tiles)
            n = int(counts.item())
        else:
            batch = nat.StrokeBatch([layer.data], [layer.mask], [ed], "cuda").upload(strokes, np.zeros(K, np.int64), labels)
            n = int(ml.select_sphere_batch(surf, batch, cull=(mode == "batch-culled"))[0])
        planes[mode] = (n, _checksum(layer.data), _checksum(layer.mask.view(torch.uint8)), _checksum(ed), layer)
    assert planes["sequential"][:4] == planes["batch-culled"][:4] == planes["batch-streamed"][:4]
    layer = planes["sequential"][4]
    assert planes["sequential"][0] == layer.valid_texels() > 0
    total = ml.layer_area(layer, surf)
    la, lc = ml.label_area(layer, surf)
    assert lc.sum() == layer.valid_texels() and abs(la.sum() - total) <= 1e-6 * total
    assert 0.0 < total <= ml.mesh_surface_area(mesh) * (1.0 + 1e-3)


# ------------------------------------------------------------------ C4

def test_config4_64_layers_batched_strokes_and_area_statistics():
    """C4: 16384^2 atlas, 64 uint8 layers, 64 batched strokes (one per layer) in ONE pass and the
    64 per-layer areas in one fused reduction: == per-layer sequential strokes / single-layer
    areas; label area and layer statistics agree with the counts."""
    import torch
    A, L = 16384, 64
    mesh = synth.heightfield_mesh(707, margin=0.01)
    surf = ml.build_surface_map(mesh, A, A)
    pool = ml.TexturePool(budget_texels=(2 * L + 8) * A * A)
    layers = [ml.create_layer("L%d" % i, "uint8", A, A, pool=pool) for i in range(L)]
    edited = [torch.zeros((A, A), dtype=torch.uint8, device="cuda") for _ in range(L)]
    strokes, labels = synth.sphere_strokes(mesh, L, seed=44, rmin_frac=0.01, rmax_frac=0.05)
    batch = nat.StrokeBatch([l.data for l in layers], [l.mask for l in layers], edited, "cuda")
    batch.upload(strokes, np.arange(L), labels)
    counts = ml.select_sphere_batch(surf, batch).cpu().numpy()
    assert (counts > 0).all()
    areas, texels = ml.layers_area(layers, surf)
    assert np.array_equal(texels, counts)
    probe = ml.create_layer("probe", "uint8", A, A, pool=pool)
    ped = torch.zeros((A, A), dtype=torch.uint8, device="cuda")
    for i in (0, 17, 63):
        probe.data.zero_(); probe.mask.zero_(); ped.zero_()
        r = ml.select_sphere(surf, probe, strokes[i, :3], strokes[i, 3], int(labels[i]), edited=ped, cull=False)
        assert r.edited_count == counts[i]
        assert _checksum(probe.data) == _checksum(layers[i].data) and _checksum(ped) == _checksum(edited[i])
        assert abs(ml.layer_area(probe, surf) - areas[i]) <= 1e-9 * areas[i]
        cnt, total, lo, hi = ml.layer_stats(layers[i])
        assert cnt == counts[i] and lo == hi == int(labels[i]) and total == int(labels[i]) * counts[i]
        la, lc = ml.label_area(layers[i], surf)
        assert lc[int(labels[i])] == counts[i] and abs(la[int(labels[i])] - areas[i]) <= 1e-9 * areas[i]


# ------------------------------------------------------------------ C5

def test_config5_32k_atlas_10m_triangles_row_slabs():
    """C5: 32768^2 atlas (1 Gtexel), 9,999,392-triangle heightfield, row-sharded.  The full map fits
    one B200 (38.7 GB), so the slabs a 2 / 4 / 8-rank job would build are compared with the rows of
    the full map; strokes and partial areas per slab add up to the full-map result (what the NCCL
    all-reduce sums)."""
    import torch
    A = 32768
    mesh = synth.heightfield_mesh(2236, margin=0.01)
    assert mesh.num_triangles == 9999392
    full = ml.build_surface_map(mesh, A, A)
    assert full.overlap == 0 and full.covered > 0.9 * A * A
    strokes, labels = synth.sphere_strokes(mesh, 4, seed=55, rmin_frac=0.01, rmax_frac=0.05)
    pool = ml.TexturePool(budget_texels=6 * A * A)
    layer = ml.create_layer("full", "uint8", A, A, pool=pool)
    n_full = sum(ml.select_sphere(full, layer, strokes[k, :3], strokes[k, 3], int(labels[k])).edited_count for k in range(4))
    area_full = ml.layer_area(layer, full)
    for world in (2, 8):
        covered = n_slabs = 0
        area_parts = 0.0
        ranks = range(world) if world == 2 else (0, 3, 7)               # every rank at 2, a sample at 8
        for rank in ranks:
            r0, rows = sharding.shard_rows(A, world, rank)
            part = ml.build_surface_map(mesh, A, A, row0=r0, rows=rows)
            assert _checksum(part.tri_id) == _checksum(full.tri_id[r0:r0 + rows])
            assert _checksum(part.pos.view(torch.int32)) == _checksum(full.pos[:, r0:r0 + rows].contiguous().view(torch.int32))
            assert _checksum(part.area.view(torch.int32)) == _checksum(full.area[r0:r0 + rows].contiguous().view(torch.int32))
            sl = ml.create_layer("slab", "uint8", A, rows, pool=pool)
            n_slabs += sum(ml.select_sphere(part, sl, strokes[k, :3], strokes[k, 3], int(labels[k])).edited_count for k in range(4))
            assert _checksum(sl.data) == _checksum(layer.data[r0:r0 + rows])
            area_parts += ml.layer_area(sl, part)
            covered += part.covered
            sl.release()
            del part
            torch.cuda.empty_cache()
        if world == 2:
            assert covered == full.covered and n_slabs == n_full
            assert abs(area_parts - area_full) <= 1e-9 * area_full
