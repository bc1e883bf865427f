#!/usr/bin/env python
"""Time the drop-in host-buffer twins (numpy planes in pageable host memory, the reference's call shape
KN:84 / KN:135-136) on the bench workload: 999,698-triangle mesh, 16384^2 atlas, r = 70 px tool.

    python tools/hostcall_time.py [--atlas 16384] [--reps 5] [--f32] [--json out.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2501_14807_b200 as ml
    from paper_2501_14807_b200 import _native as nat
    import bench as B
    ap = argparse.ArgumentParser()
    ap.add_argument("--atlas", type=int, default=16384)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--f32", action="store_true", help="float32 triangle arrays (half the upload)")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    wl = B.Workload(argparse.Namespace(atlas=a.atlas, layers=8, quads=707, window=1024), 1)
    A = a.atlas
    dt = np.float32 if a.f32 else np.float64
    tri_xy = np.ascontiguousarray(wl.mesh.tri_uv_texels(A, A), dtype=dt)
    clip = np.ascontiguousarray(wl.cam.clip_coords(wl.mesh.vertices)[wl.mesh.triangles], dtype=dt)
    depth = ml.render_depth(wl.mesh, wl.cam).plane.cpu().numpy()
    shape = np.ascontiguousarray(wl.tool_shape).astype(np.uint8)
    inp = wl.step_inputs(0)
    tool = ml.EditingTool(px=float(inp["tool_xy"][0]), py=float(inp["tool_xy"][1]), shape=shape, value=7)
    sfx, sfy, bx, by = ml.compute_tool_projection(wl.cam, tool).kernel_factors
    data, mask, edited = (np.zeros((A, A), np.uint8) for _ in range(3))
    res = {"atlas": A, "triangles": int(tri_xy.shape[0]), "tri_dtype": str(np.dtype(dt))}
    ts = []
    for r in range(a.reps + 1):
        edited[:] = 0
        t0 = time.perf_counter()
        got = nat.raster_tea(tri_xy, clip, float(wl.cam.width), float(wl.cam.height), depth, wl.eps, sfx, sfy, bx, by,
                             shape, data, mask, edited, 7)
        ts.append((time.perf_counter() - t0) * 1e3)
    res["raster_tea_ms"] = [round(t, 2) for t in ts]
    res["raster_tea_counts"] = [int(got[0]), int(got[1])]
    res["raster_tea_naive_bytes"] = int(tri_xy.nbytes + clip.nbytes + depth.nbytes + shape.nbytes + 6 * data.nbytes)
    cov = np.zeros((A, A), np.uint8)
    ts = []
    for r in range(a.reps + 1):
        cov[:] = 0
        t0 = time.perf_counter()
        w = nat.coverage_fill(tri_xy, A, A, cov)
        ts.append((time.perf_counter() - t0) * 1e3)
    res["coverage_fill_ms"] = [round(t, 2) for t in ts]
    res["coverage_written"] = int(w)
    # parity of the host call with the resident pipeline
    surf = ml.build_surface_map(wl.mesh, A, A)
    res["coverage_equals_surface_map"] = bool(w == surf.covered and np.array_equal(cov != 0, surf.coverage.cpu().numpy()))
    print(json.dumps(res, indent=1))
    if a.json:
        with open(a.json, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
