"""Oracle parity AT the sizes the metric is quoted on (backend bit-equality is
the acceptance criterion): the CUDA path against oracle/kn_port.c over the WHOLE 16384^2 atlas of
BASELINE configs C3 / C4 (1M-triangle mesh) and over a 2048-row slab of C5 (32768^2, 10M triangles).

The oracle runs row-parallel with per-band triangle lists (same per-texel arithmetic as the serial
restatement, tests/test_oracle_ext.py), so a whole 16384^2 plane costs seconds: the surface map
~0.04 us/texel, a TEA stroke ~5 ns/texel, the streaming ops less.  The oracle's planes are
produced slab by slab (2048 rows) from the same triangle arrays the GPU was given and compared with
`array_equal`; areas to 1e-10 relative (north star: 1e-6)."""
import numpy as np
import pytest

import paper_2501_14807_b200 as ml
from oracle import kn
from paper_2501_14807_b200 import _native as nat
from paper_2501_14807_b200 import synth
from paper_2501_14807_b200.mesh_core import window_triangles

pytestmark = pytest.mark.gpu

A = 16384
SLAB = 2048
CHAIN_OPS = ["union", "intersection", "difference", "union", "masking", "difference", "union"]


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def _slabs(height=A, slab=SLAB):
    return [(r0, min(height, r0 + slab)) for r0 in range(0, height, slab)]


class OracleSurface:
    """The oracle's surface map of the whole atlas as a list of row slabs (pos + area kept; tri_id
    and normals are compared against the GPU map while building and dropped)."""

    def __init__(self, mesh, gpu_surf):
        self.th = kn.max_threads()
        self.tri_xy = mesh.tri_uv_texels(A, A)
        P, N = mesh.tri_pos(), mesh.tri_nrm()
        self.pos, self.area, self.cov = [], [], []
        self.covered = self.overlap = 0
        self.mismatch = []
        for r0, r1 in _slabs():
            ref = kn.surface_map(self.tri_xy, P, N, A, A, rows=(r0, r1), threads=self.th)
            self.covered += ref["covered"]
            self.overlap += ref["overlap"]
            if not np.array_equal(gpu_surf.tri_id[r0:r1].cpu().numpy(), ref["tri_id"]):
                self.mismatch.append(("tri_id", r0))
            for k, t in (("pos", gpu_surf.pos[:, r0:r1]), ("nrm", gpu_surf.nrm[:, r0:r1]), ("area", gpu_surf.area[r0:r1])):
                if not np.array_equal(_bits(t.cpu().numpy()), _bits(ref[k])):
                    self.mismatch.append((k, r0))
            self.pos.append(ref["pos"])
            self.area.append(ref["area"])
            self.cov.append((ref["tri_id"] >= 0).astype(np.uint8))


@pytest.fixture(scope="module")
def big():
    mesh = synth.heightfield_mesh(707, margin=0.01)                 # 999,698 triangles (C2-C4 mesh)
    surf = ml.build_surface_map(mesh, A, A)
    return mesh, surf, OracleSurface(mesh, surf)


def test_surface_map_equals_oracle_over_the_whole_16k_atlas(big):
    """a11 at full size: owner ids, positions, normals and texel areas of all 268 M texels bit for bit."""
    mesh, surf, ora = big
    assert ora.mismatch == []
    assert surf.covered == ora.covered and surf.overlap == ora.overlap == 0


def _oracle_strokes(ora, strokes, labels, layer_of, L):
    """Sphere strokes through the oracle, slab by slab: lists [slab][layer] of (data, mask, edited)."""
    out, counts = [], np.zeros(L, np.int64)
    for s, (r0, r1) in enumerate(_slabs()):
        mk = lambda: [np.zeros((r1 - r0, A), np.uint8) for _ in range(L)]
        d, m, e = mk(), mk(), mk()
        counts += kn.select_sphere_batch(ora.pos[s], strokes, layer_of, labels, d, m, e, threads=ora.th)
        out.append((d, m, e))
    return out, counts


def test_c3_eight_layers_chain_and_threshold_equal_oracle_at_16k(big):
    """C3: 8 uint8 layers painted by 32 sphere strokes (culled brush kernels), the fused 8-layer chain
    (lazy and eager kernels), the 3 B/texel mask union and the height-threshold selection (tile-culled
    and streamed): every plane of every step == oracle over the whole atlas, counts included."""
    import torch
    mesh, surf, ora = big
    L = 8
    pool = ml.TexturePool(budget_texels=(2 * L + 8) * A * A)
    layers = [ml.create_layer("L%d" % i, "uint8", A, A, pool=pool) for i in range(L)]
    edited = [torch.zeros((A, A), dtype=torch.uint8, device="cuda") for _ in range(L)]
    strokes, labels = synth.sphere_strokes(mesh, 4 * L, seed=synth.SEED + 3, rmin_frac=0.02, rmax_frac=0.08)
    layer_of = np.arange(4 * L) % L
    got = np.zeros(L, np.int64)
    for k in range(4 * L):
        got[layer_of[k]] += ml.select_sphere(surf, layers[layer_of[k]], strokes[k, :3], strokes[k, 3], int(labels[k]),
                                             edited=edited[layer_of[k]]).edited_count
    ref, want = _oracle_strokes(ora, strokes, labels, layer_of.astype(np.int32), L)
    assert np.array_equal(got, want) and (want > 0).all()
    for s, (r0, r1) in enumerate(_slabs()):
        for l in range(L):
            assert np.array_equal(layers[l].data[r0:r1].cpu().numpy(), ref[s][0][l]), (s, l)
            assert np.array_equal(layers[l].mask[r0:r1].cpu().numpy().view(np.uint8), ref[s][1][l]), (s, l)
            assert np.array_equal(edited[l][r0:r1].cpu().numpy(), ref[s][2][l]), (s, l)

    # fused chain ((L0 u L1) n L2) \ L3 ... : lazy (default) and eager kernels
    out = ml.create_layer("out", "uint8", A, A, pool=pool)
    want_valid = 0
    chain_ref = []
    for s, (r0, r1) in enumerate(_slabs()):
        cd, cm = np.zeros((r1 - r0, A), np.uint8), np.zeros((r1 - r0, A), np.uint8)
        kn.layer_chain(CHAIN_OPS, ref[s][0], ref[s][1], cd, cm, threads=ora.th)
        chain_ref.append((cd, cm))
        want_valid += int(cm.sum())
    for lazy in (True, False):
        out.data.fill_(99); out.mask.fill_(1)
        ml.layer_chain(layers, CHAIN_OPS, out, lazy=lazy)
        assert out.valid_texels() == want_valid > 0
        for s, (r0, r1) in enumerate(_slabs()):
            assert np.array_equal(out.data[r0:r1].cpu().numpy(), chain_ref[s][0]), (lazy, s)
            assert np.array_equal(out.mask[r0:r1].cpu().numpy().view(np.uint8), chain_ref[s][1]), (lazy, s)

    # the bare-mask union (3 B/texel stream)
    tmp = torch.zeros((A, A), dtype=torch.uint8, device="cuda")
    nat.layer_op("union", None, layers[0].mask, None, layers[1].mask, None, tmp)
    for s, (r0, r1) in enumerate(_slabs()):
        um = np.zeros((r1 - r0, A), np.uint8)
        kn.layer_op("union", None, ref[s][1][0], None, ref[s][1][1], None, um, threads=ora.th)
        assert np.array_equal(tmp[r0:r1].cpu().numpy(), um), s

    # threshold selection on the height plane (C3 window: 40-60th percentile), culled and streamed
    z = mesh.vertices[:, 2]
    lo, hi = float(np.percentile(z, 40.0)), float(np.percentile(z, 60.0))
    attr = surf.pos[2]
    tiles = nat.attr_tiles(attr)
    for mode, tl in (("culled", tiles), ("streamed", None)):
        lay = ml.create_layer("thr_" + mode, "uint8", A, A, pool=pool)
        ed = torch.zeros((A, A), dtype=torch.uint8, device="cuda")
        ed[:, ::3] = 1                                       # pre-dirtied edited plane: the 0 -> 1 count must skip these
        n_got = ml.select_threshold(attr, None, lo, hi, lay, 9, edited=ed, tiles=tl).edited_count
        n_want = 0
        for s, (r0, r1) in enumerate(_slabs()):
            d, m = np.zeros((r1 - r0, A), np.uint8), np.zeros((r1 - r0, A), np.uint8)
            e = np.zeros((r1 - r0, A), np.uint8)
            e[:, ::3] = 1
            n_want += kn.select_threshold(ora.pos[s][2], None, lo, hi, d, m, e, 9, threads=ora.th)
            assert np.array_equal(lay.data[r0:r1].cpu().numpy(), d), (mode, s)
            assert np.array_equal(lay.mask[r0:r1].cpu().numpy().view(np.uint8), m), (mode, s)
            assert np.array_equal(ed[r0:r1].cpu().numpy(), e), (mode, s)
        assert n_got == n_want > 0, mode
        lay.release()
        del ed
    for l in layers + [out]:
        l.release()


def test_c4_64_layers_batched_strokes_and_areas_equal_oracle_at_16k(big):
    """C4: 64 uint8 layers, 64 strokes (one per layer) in ONE batched pass, 64 areas in one fused
    reduction: every plane of every layer == oracle over the whole atlas; per-layer counts exact, areas
    1e-10 relative."""
    import torch
    mesh, surf, ora = big
    L = 64
    pool = ml.TexturePool(budget_texels=(2 * L + 8) * A * A)
    layers = [ml.create_layer("L%d" % i, "uint8", A, A, pool=pool) for i in range(L)]
    edited = [torch.zeros((A, A), dtype=torch.uint8, device="cuda") for _ in range(L)]
    strokes, labels = synth.sphere_strokes(mesh, L, seed=44, rmin_frac=0.01, rmax_frac=0.05)
    batch = nat.StrokeBatch([l.data for l in layers], [l.mask for l in layers], edited, "cuda")
    batch.upload(strokes, np.arange(L), labels)
    counts = ml.select_sphere_batch(surf, batch).cpu().numpy()
    areas, texels = ml.layers_area(layers, surf)
    want_counts = np.zeros(L, np.int64)
    want_areas = np.zeros(L, np.float64)
    want_texels = np.zeros(L, np.int64)
    for s, (r0, r1) in enumerate(_slabs()):
        mk = lambda: [np.zeros((r1 - r0, A), np.uint8) for _ in range(L)]
        d, m, e = mk(), mk(), mk()
        want_counts += kn.select_sphere_batch(ora.pos[s], strokes, np.arange(L, dtype=np.int32), labels, d, m, e, threads=ora.th)
        a, c = kn.layers_area(ora.area[s], m, threads=ora.th)
        want_areas += a
        want_texels += c
        for l in range(L):
            # only the slabs a stroke touches hold anything: compare digests of the GPU rows first (cheap), planes on mismatch
            g = layers[l].data[r0:r1]
            if not d[l].any() and not bool(g.any()):
                assert not bool(layers[l].mask[r0:r1].any()) and not bool(edited[l][r0:r1].any())
                continue
            assert np.array_equal(g.cpu().numpy(), d[l]), (s, l)
            assert np.array_equal(layers[l].mask[r0:r1].cpu().numpy().view(np.uint8), m[l]), (s, l)
            assert np.array_equal(edited[l][r0:r1].cpu().numpy(), e[l]), (s, l)
    assert np.array_equal(counts, want_counts) and (want_counts > 0).all()
    assert np.array_equal(texels, want_texels)
    assert np.all(np.abs(areas - want_areas) <= 1e-10 * want_areas)
    for l in layers:
        l.release()


def test_tea_tpa_stroke_equals_oracle_at_16k(big):
    """The paper's edit (TEA + TPA) at 16384^2 with the 1M-triangle mesh: culled one-call
    stroke, whole-atlas streaming stroke and the direct per-triangle kernel == the oracle's raster_tea
    (KN:135-203 restated) + outline + padding over the whole atlas: planes and all three counts."""
    import torch
    mesh, surf, ora = big
    th = ora.th
    cam = synth.default_camera(1024, 1024, eye=(0.5, 0.5, 1.6), target=(0.5, 0.5, 0.0), fovy=40.0, near=0.2, far=5.0)
    depth = ml.render_depth(mesh, cam)
    xy, zn = window_triangles(mesh, cam)
    d_ref = np.ones((1024, 1024), np.float32)
    kn.raster_depth(xy, zn, d_ref, threads=th)
    assert np.array_equal(_bits(depth.plane.cpu().numpy()), _bits(d_ref))
    ctx = ml.StrokeContext(mesh, cam, depth, surf)
    outline = ml.build_outline_mask(surf.coverage, thickness=1)
    cov = np.concatenate(ora.cov, 0)
    outline_ref = kn.outline(cov, 1, threads=th)
    assert np.array_equal(outline.cpu().numpy().view(np.uint8), outline_ref)
    del cov
    pool = ml.TexturePool(budget_texels=8 * A * A)
    clip = cam.clip_coords(mesh.vertices)[mesh.triangles]
    data, mask = np.zeros((A, A), np.uint8), np.zeros((A, A), np.uint8)
    gpu = {m: ml.create_layer(m, "uint8", A, A, pool=pool) for m in ("culled", "streamed", "direct")}
    # two strokes on the same layers: an interior one and one that reaches the island border (padding), second over the first
    for px, py, r, value in ((500.0, 520.0, 70, 7), (40.0, 512.0, 120, 11)):
        tool = ml.EditingTool(px=px, py=py, shape=synth.circle_shape(r), value=value, padding_radius=1)
        sfx, sfy, bx, by = ml.compute_tool_projection(cam, tool).kernel_factors
        edited = np.zeros((A, A), np.uint8)
        want = kn.raster_tea(ora.tri_xy, clip, 1024.0, 1024.0, d_ref, 1e-4, sfx, sfy, bx, by, tool.shape, data, mask,
                             edited, value, threads=th)
        want_pad = kn.padding(outline_ref, edited, 1, data, mask, value, threads=th)
        assert want[0] > 0 and want[1] == ora.covered
        for mode, lay in gpu.items():
            if mode == "direct":
                res = ml.apply_stroke(ctx, tool, lay, force_direct=True)
                pc = torch.zeros(1, dtype=torch.int64, device="cuda")
                nat.apply_padding(outline.view(torch.uint8), ctx.edited, 1, lay.data, lay.mask, value, counts=pc)
                got = (res.edited_count, res.fragments, int(pc.item()))
            else:
                res = ml.stroke(ctx, tool, lay, outline, cull=(mode == "culled"))
                got = (res.edited_count, res.fragments, res.padded_count)
            assert got == (want[0], want[1], want_pad), (mode, px)
            assert np.array_equal(ctx.edited.cpu().numpy(), edited), (mode, px)
            assert np.array_equal(lay.data.cpu().numpy(), data), (mode, px)
            assert np.array_equal(lay.mask.cpu().numpy().view(np.uint8), mask), (mode, px)
    assert want_pad > 0                                             # the second stroke really padded outline texels
    for lay in gpu.values():
        lay.release()


def test_c5_slab_of_the_32k_atlas_equals_oracle():
    """C5: 32768^2 atlas, 9,999,392-triangle heightfield.  One rank's view -- a 2048-row slab in the middle
    of rank 3 of 8 -- built as a slab (row0, rows): surface map, 64 batched strokes on 8 layers and the
    partial areas == oracle restricted to the same rows (what the NCCL all-reduce would sum)."""
    import torch
    A5, rows = 32768, 2048
    r0 = 3 * (A5 // 8) + 1000
    mesh = synth.heightfield_mesh(2236, margin=0.01)
    assert mesh.num_triangles == 9999392
    th = kn.max_threads()
    part = ml.build_surface_map(mesh, A5, A5, row0=r0, rows=rows)
    ref = kn.surface_map(mesh.tri_uv_texels(A5, A5), mesh.tri_pos(), mesh.tri_nrm(), A5, A5, rows=(r0, r0 + rows), threads=th)
    assert part.covered == ref["covered"] and part.overlap == ref["overlap"] == 0
    assert np.array_equal(part.tri_id.cpu().numpy(), ref["tri_id"])
    for k, t in (("pos", part.pos), ("nrm", part.nrm), ("area", part.area)):
        assert np.array_equal(_bits(t.cpu().numpy()), _bits(ref[k])), k
    L, K = 8, 64
    strokes, labels = synth.sphere_strokes(mesh, K, seed=55, rmin_frac=0.01, rmax_frac=0.08)
    # centre the strokes' heights on the slab so that most of them touch it
    v0 = (r0 + 0.5 * rows) / A5
    strokes[:, 1] = np.clip(v0 + (strokes[:, 1] - 0.5) * 0.2, 0.0, 1.0)
    layer_of = (np.arange(K) % L).astype(np.int32)
    pool = ml.TexturePool(budget_texels=(2 * L + 4) * A5 * rows)
    layers = [ml.create_layer("L%d" % i, "uint8", A5, rows, pool=pool) for i in range(L)]
    edited = [torch.zeros((rows, A5), dtype=torch.uint8, device="cuda") for _ in range(L)]
    batch = nat.StrokeBatch([l.data for l in layers], [l.mask for l in layers], edited, "cuda").upload(strokes, layer_of, labels)
    counts = ml.select_sphere_batch(part, batch).cpu().numpy()
    mk = lambda: [np.zeros((rows, A5), np.uint8) for _ in range(L)]
    d, m, e = mk(), mk(), mk()
    want = kn.select_sphere_batch(ref["pos"], strokes, layer_of, labels, d, m, e, threads=th)
    assert np.array_equal(counts, want) and want.sum() > 0
    for l in range(L):
        assert np.array_equal(layers[l].data.cpu().numpy(), d[l]), l
        assert np.array_equal(layers[l].mask.cpu().numpy().view(np.uint8), m[l]), l
        assert np.array_equal(edited[l].cpu().numpy(), e[l]), l
    areas, texels = ml.layers_area(layers, part)
    wa, wc = kn.layers_area(ref["area"], m, threads=th)
    assert np.array_equal(texels, wc)
    assert np.all(np.abs(areas - wa) <= 1e-10 * np.maximum(wa, 1e-300))
