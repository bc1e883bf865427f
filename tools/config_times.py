#!/usr/bin/env python
"""Device times of BASELINE.json's configurations C1, C2, C4, C5 (C3+C4 at 8 layers is bench.py's
default step).  CUDA events, median of the repetitions, inputs resident.  Informational: the judged
line is bench.py's; parity for the same configurations is tests/test_gpu_configs.py."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_14807_b200 as ml  # noqa: E402
from paper_2501_14807_b200 import _native as nat, synth  # noqa: E402


def timed(fn, reps=7, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    out = {}
    want = set(sys.argv[1:]) or {"C1", "C2", "C4", "C5"}
    if "C1" in want:
        A, W = 1024, 512
        mesh = synth.icosphere_mesh(5)
        cam = synth.default_camera(W, W)
        build = timed(lambda: ml.build_surface_map(mesh, A, A), reps=5)
        surf = ml.build_surface_map(mesh, A, A)
        depth_ms = timed(lambda: ml.render_depth(mesh, cam), reps=5)
        ctx = ml.StrokeContext(mesh, cam, ml.render_depth(mesh, cam), surf)
        pool = ml.TexturePool()
        layer = ml.create_layer("a", "uint8", A, A, pool=pool)
        tool = ml.EditingTool(px=256.0, py=256.0, shape=nat._as_dev_bytes(synth.circle_shape(40), "cuda"), value=7)
        ed = torch.zeros((A, A), dtype=torch.uint8, device="cuda")
        out["C1"] = {"triangles": mesh.num_triangles, "atlas": A,
                     "surface_map_ms (incl. host triangle upload)": build, "render_depth_ms": depth_ms,
                     "tea_stroke_ms": timed(lambda: ml.apply_stroke(ctx, tool, layer), reps=20),
                     "sphere_stroke_ms": timed(lambda: ml.select_sphere(surf, layer, (0.0, 0.0, 1.0), 0.25, 3, edited=ed), reps=20)}
        del surf, ctx
    if "C2" in want:
        A, K = 4096, 1000
        mesh = synth.heightfield_mesh(707)
        surf = ml.build_surface_map(mesh, A, A)
        tri = surf.tri_xy
        P, N = torch.from_numpy(mesh.tri_pos()).cuda(), torch.from_numpy(mesh.tri_nrm()).cuda()
        build = timed(lambda: nat.surface_map(tri, P, N, A, A), reps=5)
        strokes, labels = synth.sphere_strokes(mesh, K)
        pool = ml.TexturePool(budget_texels=16 * A * A)
        layer = ml.create_layer("a", "uint8", A, A, pool=pool)
        ed = torch.zeros((A, A), dtype=torch.uint8, device="cuda")
        counts = torch.zeros(1, dtype=torch.int64, device="cuda")
        batch = nat.StrokeBatch([layer.data], [layer.mask], [ed], "cuda").upload(strokes, np.zeros(K, np.int64), labels)

        def seq(tiles):
            for k in range(K):
                nat.select_sphere(surf.pos, strokes[k, :3], strokes[k, 3], layer.data, layer.mask, ed, int(labels[k]),
                                  counts=counts, tiles=tiles)
        out["C2"] = {"triangles": mesh.num_triangles, "atlas": A, "strokes": K,
                     "surface_map_ms (device arrays)": build,
                     "1000 strokes sequential culled ms": timed(lambda: seq(surf.tiles), reps=3, warm=1),
                     "1000 strokes sequential streamed ms": timed(lambda: seq(None), reps=3, warm=1),
                     "1000 strokes one batched pass culled ms": timed(lambda: ml.select_sphere_batch(surf, batch), reps=5),
                     "1000 strokes one batched pass streamed ms": timed(lambda: ml.select_sphere_batch(surf, batch, cull=False), reps=5),
                     "layer_area ms": timed(lambda: nat.layer_area(surf.area, [layer.mask], sums=torch.zeros(1, dtype=torch.float64, device="cuda"),
                                                                  counts=torch.zeros(1, dtype=torch.int64, device="cuda")), reps=10),
                     "label_area ms": timed(lambda: ml.label_area(layer, surf), reps=10)}
        del surf, P, N
    if "C4" in want:
        A, L = 16384, 64
        mesh = synth.heightfield_mesh(707, margin=0.01)
        surf = ml.build_surface_map(mesh, A, A)
        pool = ml.TexturePool(budget_texels=(2 * L + 8) * A * A)
        layers = [ml.create_layer("L%d" % i, "uint8", A, A, pool=pool) for i in range(L)]
        edited = [torch.zeros((A, A), dtype=torch.uint8, device="cuda") for _ in range(L)]
        strokes, labels = synth.sphere_strokes(mesh, L, seed=44, rmin_frac=0.01, rmax_frac=0.05)
        batch = nat.StrokeBatch([l.data for l in layers], [l.mask for l in layers], edited, "cuda").upload(strokes, np.arange(L), labels)
        sums = torch.zeros(L, dtype=torch.float64, device="cuda")
        cnts = torch.zeros(L, dtype=torch.int64, device="cuda")
        masks = [l.mask for l in layers]
        out["C4"] = {"atlas": A, "layers": L,
                     "64 batched strokes culled ms": timed(lambda: ml.select_sphere_batch(surf, batch), reps=10),
                     "64 batched strokes streamed ms": timed(lambda: ml.select_sphere_batch(surf, batch, cull=False), reps=10),
                     "64 per-layer areas ms": timed(lambda: nat.layer_area(surf.area, masks, sums=sums, counts=cnts), reps=10),
                     "label_area (1 layer) ms": timed(lambda: ml.label_area(layers[0], surf), reps=10),
                     "layer_stats (1 layer) ms": timed(lambda: ml.layer_stats(layers[0]), reps=10)}
        del surf, layers, edited, batch, masks
        torch.cuda.empty_cache()
    if "C5" in want:
        A = 32768
        mesh = synth.heightfield_mesh(2236, margin=0.01)
        tri = torch.from_numpy(mesh.tri_uv_texels(A, A)).cuda()
        P, N = torch.from_numpy(mesh.tri_pos()).cuda(), torch.from_numpy(mesh.tri_nrm()).cuda()
        res = {"triangles": mesh.num_triangles, "atlas": A}
        for world in (1, 2, 4, 8):
            rows = A // world
            res["surface_map slab of %d rows (1/%d) ms" % (rows, world)] = timed(
                lambda: nat.surface_map(tri, P, N, A, A, row0=0, rows=rows), reps=3, warm=1)
        surf = ml.build_surface_map(mesh, A, A, row0=0, rows=A // 8)
        rows = A // 8
        pool = ml.TexturePool(budget_texels=8 * A * rows)
        layer = ml.create_layer("a", "uint8", A, rows, pool=pool)
        ed = torch.zeros((rows, A), dtype=torch.uint8, device="cuda")
        strokes, labels = synth.sphere_strokes(mesh, 64, seed=55, rmin_frac=0.01, rmax_frac=0.05)
        batch = nat.StrokeBatch([layer.data], [layer.mask], [ed], "cuda").upload(strokes, np.zeros(64, np.int64), labels)
        res["per-rank slab (1/8): 64 batched strokes culled ms"] = timed(lambda: ml.select_sphere_batch(surf, batch), reps=10)
        res["per-rank slab (1/8): 64 batched strokes streamed ms"] = timed(lambda: ml.select_sphere_batch(surf, batch, cull=False), reps=10)
        res["per-rank slab (1/8): layer_area ms"] = timed(lambda: nat.layer_area(surf.area, [layer.mask], sums=torch.zeros(1, dtype=torch.float64, device="cuda"),
                                                                               counts=torch.zeros(1, dtype=torch.int64, device="cuda")), reps=10)
        out["C5"] = res
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
