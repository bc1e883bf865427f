#!/usr/bin/env python
"""The paper's engine comparison (Fig 5, Fig 7, Table 1) on one B200: the texture
engine (TEA + TPA strokes) against the OCT-TR octree baseline (ray-cast edits), same mesh, camera,
tool positions and radii, matched levels (2048/4096/8192 <-> depth 11/12/13, PAPER section 5).

    python tools/octree_compare.py [--mesh terrain:707] [--out-prefix gpurun_out/octree] [--small]

Writes <prefix>_texture.csv and <prefix>_octree.csv (frozen schema) and <prefix>.json with
the medians, build times, transfer bytes, precision table, kernel rates (pairs/s, rays/s) and the CPU
restatement (oracle/kn_port.c, OpenMP) cast over the same rays for scale.  Tuning / reporting aid, not
the judged benchmark (bench.py)."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_14807_b200 as ml  # noqa: E402
from paper_2501_14807_b200 import _native as nat, bench, octree  # noqa: E402


def ev_time(fn, reps=5):
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
    ap = argparse.ArgumentParser()
    ap.add_argument("--mesh", default="terrain:707")
    ap.add_argument("--out-prefix", default=os.path.join(ROOT, "gpurun_out", "octree"))
    ap.add_argument("--small", action="store_true", help="2 levels, 3 radii (smoke run)")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    res = (1024, 2048) if args.small else (2048, 4096, 8192)
    dep = (10, 11) if args.small else (11, 12, 13)
    radii = (10, 70, 200) if args.small else (10, 40, 70, 100, 200)
    common = dict(meshes=[args.mesh], resolutions=res, depths=dep, radii=radii, repetitions=5,
                  window=(1024, 1024))
    out = {"mesh": args.mesh, "levels": list(zip(res, dep)), "radii": list(radii)}
    os.makedirs(os.path.dirname(args.out_prefix), exist_ok=True)
    for engine in ("texture", "octree"):
        plan = bench.BenchPlan(engine=engine, **common)
        t0 = time.time()
        recs = bench.run_radius_sweep(plan)
        bench.write_csv(recs, "%s_%s.csv" % (args.out_prefix, engine))
        out[engine] = [{"level": r.level, "radius": r.radius, "median_ms": r.median_ms, "cells": r.cells,
                        "transfer_bytes": r.transfer_bytes, "build_ms": r.build_ms, "peak_bytes": r.peak_bytes,
                        "outcome": r.outcome} for r in recs]
        out[engine + "_precision"] = bench.run_precision_table(plan)
        out[engine + "_wall_s"] = round(time.time() - t0, 1)
        torch.cuda.empty_cache()

    # kernel rates at the deepest level: expansion of the last level and the r=200 ray set
    mesh = bench.make_mesh(args.mesh)
    cam = bench.make_camera(args.mesh, (1024, 1024))
    d = dep[-1]
    tree = ml.build_octree(mesh, d)
    prev = ml.build_octree(mesh, d - 1)
    pc = prev.leaf_cells().to(torch.int32).contiguous()
    counts = (prev.offsets[1:] - prev.offsets[:-1])
    pp = torch.repeat_interleave(torch.arange(prev.leaf_count, device="cuda", dtype=torch.int32), counts)
    pt = prev.tri_idx
    child_h = tree.side / float(1 << d)
    ms = ev_time(lambda: nat.expand_pairs_ordered(tree.verts, tree.tris, pc, pp, pt, tree.cube_min, child_h))
    out["expand"] = {"depth": d, "pairs_in": int(pt.shape[0]), "rows_out": int(tree.tri_idx.shape[0]), "ms": ms,
                     "Mpairs_s": pt.shape[0] / ms / 1e3, "M_sat_tests_s": 8 * pt.shape[0] / ms / 1e3}
    tool = ml.EditingTool(px=512.0, py=512.0, shape=ml.synth.circle_shape(radii[-1]), value=7)
    od, dd = octree.tool_rays(cam, tool, device="cuda")
    o, dr = od.cpu().numpy(), dd.cpu().numpy()
    cast = lambda: nat.raycast(od, dd, tree.keys, tree.offsets, tree.tri_idx, tree.verts, tree.tris,  # noqa: E731
                               tree.cube_min, tree.h, tree.n_cells, tree.coarse, tree.coarse_shift, None)
    ms = ev_time(cast)
    bt, btri, leaf = cast()
    out["raycast"] = {"depth": d, "rays": len(o), "hits": int((leaf >= 0).sum().item()), "ms": ms,
                      "Mrays_s": len(o) / ms / 1e3, "leaves": tree.leaf_count, "build_ms": tree.build_ms,
                      "node_count": tree.node_count}
    if not args.no_cpu:
        sys.path.insert(0, ROOT)
        from oracle import kn
        k = tree.keys.cpu().numpy().astype(np.uint64)
        off, idx = tree.offsets.cpu().numpy(), tree.tri_idx.cpu().numpy()
        v, t = mesh.vertices, mesh.triangles
        cz = tree.coarse.cpu().numpy()
        t0 = time.perf_counter()
        cbt, cbtri, cleaf = kn.raycast(o, dr, k, off, idx, v, t, tree.cube_min, tree.h, tree.n_cells, cz,
                                       tree.coarse_shift, threads=0)
        cpu_ms = (time.perf_counter() - t0) * 1e3
        out["raycast"]["cpu_port_ms"] = cpu_ms
        out["raycast"]["cpu_threads"] = kn.max_threads()
        out["raycast"]["equal_to_cpu_port"] = bool(np.array_equal(cbt, bt.cpu().numpy())
                                                   and np.array_equal(cbtri, btri.cpu().numpy())
                                                   and np.array_equal(cleaf, leaf.cpu().numpy()))
    with open(args.out_prefix + ".json", "w") as f:
        json.dump(out, f, indent=1)
    for engine in ("texture", "octree"):
        for r in out[engine]:
            print(engine, r["level"], r["radius"], r["median_ms"], r["cells"], r["transfer_bytes"], r["outcome"])
    print(json.dumps({"expand": out["expand"], "raycast": out["raycast"]}))


if __name__ == "__main__":
    main()
