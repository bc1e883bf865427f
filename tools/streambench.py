#!/usr/bin/env python
"""Whole-atlas streaming forms of the hot-path stages on the bench workload, timed WITHOUT host
launch latency: every case is captured into a CUDA graph holding `--inner` back-to-back calls, the
graph is replayed `--reps` times and the median replay time / inner is reported.  (A single call
between two events on an idle GPU measures the host's issue latency as well -- 10-30 us of Python +
ctypes per call, a third of a 75 us kernel.)

    python tools/streambench.py [--atlas 16384] [--inner 10] [--reps 7] [--json out.json] [names...]

Prints name, ms per call, algorithmic GB/s (SURVEY.md 8(d) bytes), fraction of the measured HBM
peak (MEASURED_PEAKS.json).  Not the judged benchmark (bench.py is); the timing routine is bench.py's
`time_graph`, the one behind its `stream_kernels` block."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def time_graph(fn, inner=10, reps=7, warm=2):
    """bench.time_graph: median ms per call over replays of a CUDA graph holding `inner` back-to-back calls."""
    import bench
    return bench.time_graph(fn, inner=inner, reps=reps, warm=warm)


def main():
    import torch
    import paper_2501_14807_b200 as ml
    from paper_2501_14807_b200 import _native as nat, synth
    import bench as B

    ap = argparse.ArgumentParser()
    ap.add_argument("--atlas", type=int, default=16384)
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--inner", type=int, default=10)
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--json", default=None)
    ap.add_argument("--eager", action="store_true", help="three plain calls per case and no timing (for ncu captures)")
    ap.add_argument("names", nargs="*")
    a = ap.parse_args()
    args = argparse.Namespace(atlas=a.atlas, layers=a.layers, quads=707, window=1024)
    wl = B.Workload(args, 1)
    peak, _ = B.measured_peak()
    dev = torch.device("cuda", 0)
    W = rows = wl.A
    n = rows * W
    L = wl.L
    surf = ml.build_surface_map(wl.mesh, W, rows, device=dev)
    depth = ml.render_depth(wl.mesh, wl.cam, device=dev)
    ctx = ml.StrokeContext(wl.mesh, wl.cam, depth, surf, device=dev)
    pool = ml.TexturePool(budget_texels=(2 * L + 8) * n + 1, device=dev)
    layers = [ml.create_layer("L%d" % i, "uint8", W, rows, pool=pool) for i in range(L)]
    out_layer = ml.create_layer("out", "uint8", W, rows, pool=pool)
    edited = [torch.zeros((rows, W), dtype=torch.uint8, device=dev) for _ in range(L)]
    tmp_mask = torch.zeros((rows, W), dtype=torch.uint8, device=dev)
    outline = nat.outline_mask(surf.coverage.to(torch.uint8), 1)
    for k in range(len(wl.seed_strokes)):
        ml.select_sphere(surf, layers[k % L], wl.seed_strokes[k, :3], wl.seed_strokes[k, 3], wl.seed_labels[k], edited=edited[k % L])
    inp = wl.step_inputs(0)
    tool = ml.EditingTool(px=float(inp["tool_xy"][0]), py=float(inp["tool_xy"][1]), shape=nat._as_dev_bytes(wl.tool_shape, dev), value=7)
    batch = nat.StrokeBatch([l.data for l in layers], [l.mask for l in layers], edited, dev)
    batch.upload(inp["batch"], inp["batch_layers"], inp["batch_values"])
    attr = surf.pos[2]
    c1 = torch.zeros(1, dtype=torch.int64, device=dev)
    sums = torch.zeros(L, dtype=torch.float64, device=dev)
    cnts = torch.zeros(L, dtype=torch.int64, device=dev)
    T = wl.mesh.num_triangles
    g = torch.Generator(device=dev).manual_seed(1)
    dense = []

    def dense_masks():
        if not dense:
            for k in range(L):
                yy, xx = torch.meshgrid(torch.linspace(0, 9 + k, rows, device=dev), torch.linspace(0, 7 + k, W, device=dev), indexing="ij")
                f = torch.sin(xx + k) * torch.cos(yy - k)
                dense.append((f > 0.4).to(torch.uint8))
                del yy, xx, f
        return dense

    ml.apply_stroke(ctx, tool, layers[0], eps=wl.eps, cull=False)          # marks for the padding case
    s = inp["sphere"]
    cases = [
        ("copy 1 plane (torch, 2 B/texel)", lambda: tmp_mask.copy_(layers[0].mask), 2 * n),
        ("memset 1 plane (torch)", lambda: tmp_mask.zero_(), n),
        ("tpa stream", lambda: nat.apply_padding(outline, ctx.edited, 1, layers[0].data, layers[0].mask, 7, counts=c1), wl.algorithmic_bytes(n, "tpa", T)),
        ("tea stream (stage: reset+classify+stream+eval)", lambda: ml.apply_stroke(ctx, tool, layers[0], eps=wl.eps, cull=False), wl.algorithmic_bytes(n, "tea", T)),
        ("threshold stream", lambda: nat.select_threshold(attr, None, wl.thr[0], wl.thr[1], layers[2].data, layers[2].mask, edited[2], 9, counts=c1), 4 * n),
        ("thr-nohit stream", lambda: nat.select_threshold(attr, None, 50.0, 60.0, layers[2].data, layers[2].mask, edited[2], 9, counts=c1), 4 * n),
        ("thr-allhit stream", lambda: nat.select_threshold(attr, None, -50.0, 60.0, layers[2].data, layers[2].mask, edited[2], 9, counts=c1), 8 * n),
        ("mask_op", lambda: nat.layer_op("union", None, layers[0].mask, None, layers[1].mask, None, tmp_mask), 3 * n),
        ("layer_op union u8 (6 B/texel)", lambda: nat.layer_op("union", layers[0].data, layers[0].mask, layers[1].data, layers[1].mask, out_layer.data, out_layer.mask), 6 * n),
        ("area L=%d bench masks" % L, lambda: nat.layer_area(surf.area, [l.mask for l in layers], sums=sums, counts=cnts), wl.algorithmic_bytes(n, "area", T)),
        ("area L=%d dense masks" % L, lambda: nat.layer_area(surf.area, dense_masks(), sums=sums, counts=cnts), wl.algorithmic_bytes(n, "area", T)),
        ("area L=1", lambda: nat.layer_area(surf.area, [layers[0].mask], sums=sums[:1], counts=cnts[:1]), 5 * n),
        ("chain eager", lambda: ml.layer_chain(layers[:wl.chain_n], wl.chain_ops, out_layer, lazy=False), wl.algorithmic_bytes(n, "chain", T)),
        ("chain lazy", lambda: ml.layer_chain(layers[:wl.chain_n], wl.chain_ops, out_layer, lazy=True), wl.algorithmic_bytes(n, "chain", T)),
        ("sphere stream", lambda: nat.select_sphere(surf.pos, s[:3], s[3], layers[1].data, layers[1].mask, edited[1], 3, counts=c1), 12 * n),
        ("batch stream", lambda: nat.select_sphere_batch(surf.pos, batch), 12 * n),
    ]
    res = {}
    for name, fn, nbytes in cases:
        if a.names and not any(w in name for w in a.names):
            continue
        if "dense" in name:
            dense_masks()
        if a.eager:
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            continue
        ms, graphed = time_graph(fn, a.inner, a.reps)
        gbs = nbytes / ms / 1e6
        res[name] = {"ms": round(ms, 4), "gb_s": round(gbs, 1), "frac_of_peak": round(gbs / peak, 4), "graph": graphed}
        print("%-48s %8.4f ms  %8.1f GB/s  %6.3f of %.0f  %s" % (name, ms, gbs, gbs / peak, peak, "graph" if graphed else "eager"), flush=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
