#!/usr/bin/env python
"""Kernel micro-benchmarks on synthetic planes (no mesh needed): quick A/B timing while tuning.

    python tools/microbench.py [--n 16384] [--reps 20] [names...]

Prints one line per case: name, ms (median of reps, CUDA events), GB/s of the bytes given.
Not a parity test and not the judged benchmark (that is bench.py)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_14807_b200 import _native as nat  # noqa: E402


def timeit(fn, reps):
    for _ in range(3):
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
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("names", nargs="*")
    args = ap.parse_args()
    N = args.n
    n = N * N
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(1)
    want = set(args.names)

    def run(name, fn, nbytes):
        if want and not any(w in name for w in want):
            return
        ms = timeit(fn, args.reps)
        print("%-34s %8.4f ms  %8.1f GB/s  %8.1f Gtexel/s" % (name, ms, nbytes / ms / 1e6, n / ms / 1e6), flush=True)

    if not want or any("raster" in w for w in want):
        # rasteriser: C2 mesh (999,698 triangles) into 4096^2 and 16384^2 atlases; Mtri/s
        from paper_2501_14807_b200 import synth, mesh_core
        import paper_2501_14807_b200 as ml
        mesh = synth.heightfield_mesh(707, margin=0.01)
        cam = synth.default_camera(1024, 1024, eye=(0.5, 0.5, 1.6), target=(0.5, 0.5, 0.0), fovy=40.0, near=0.2, far=5.0)
        T = mesh.num_triangles
        for A in (4096, 16384):
            xy = torch.from_numpy(mesh.tri_uv_texels(A, A)).to(dev)
            P, Nn = torch.from_numpy(mesh.tri_pos()).to(dev), torch.from_numpy(mesh.tri_nrm()).to(dev)
            cov = torch.zeros((A, A), dtype=torch.uint8, device=dev)
            c2 = torch.zeros(2, dtype=torch.int64, device=dev)
            for nm, fn in (("raster coverage_fill", lambda: nat.coverage_fill(xy, A, A, cov, counts=c2)),
                           ("raster surface_map (id+resolve)", lambda: nat.surface_map(xy, P, Nn, A, A))):
                ms = timeit(fn, 5)
                print("%-34s %8.3f ms  %8.1f Mtri/s  %8.2f Gtexel/s  (atlas %d^2)" % (nm, ms, T / ms / 1e3, A * A / ms / 1e6, A), flush=True)
            clip = torch.from_numpy(np.ascontiguousarray(cam.clip_coords(mesh.vertices)[mesh.triangles])).to(dev)
            depth = ml.render_depth(mesh, cam)
            shape = nat._as_dev_bytes(synth.circle_shape(70), dev)
            d = torch.zeros((A, A), dtype=torch.uint8, device=dev)
            m = torch.zeros((A, A), dtype=torch.uint8, device=dev)
            e = torch.zeros((A, A), dtype=torch.uint8, device=dev)
            ms = timeit(lambda: nat.raster_tea(xy, clip, 1024.0, 1024.0, depth.plane, 1e-4, 3.66, 3.66, 0.5, 0.5, shape,
                                               d, m, e, 7, counts=c2), 5)
            print("%-34s %8.3f ms  %8.1f Mtri/s  %8.2f Gtexel/s  (atlas %d^2)" % ("raster_tea direct (KN:135)", ms, T / ms / 1e3, A * A / ms / 1e6, A), flush=True)
            del xy, P, Nn, cov, clip, d, m, e
        wxy, wzn = mesh_core.window_triangles(mesh, cam)
        wxy, wzn = torch.from_numpy(wxy).to(dev), torch.from_numpy(wzn).to(dev)
        dep = torch.ones((1024, 1024), dtype=torch.float32, device=dev)
        ms = timeit(lambda: (dep.fill_(1.0), nat.raster_depth(wxy, wzn, dep)), 5)
        print("%-34s %8.3f ms  %8.1f Mtri/s  (window 1024^2)" % ("raster_depth", ms, T / ms / 1e3), flush=True)
        torch.cuda.empty_cache()

    # smooth attribute field: coherent hit regions like a real attribute
    yy, xx = torch.meshgrid(torch.linspace(0, 6, N, device=dev), torch.linspace(0, 6, N, device=dev), indexing="ij")
    attr = (torch.sin(xx) * torch.cos(yy)).contiguous()
    del yy, xx
    data = torch.zeros((N, N), dtype=torch.uint8, device=dev)
    mask = torch.zeros((N, N), dtype=torch.uint8, device=dev)
    edited = torch.zeros((N, N), dtype=torch.uint8, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    for name, lo, hi in (("threshold hits=0%", 5.0, 6.0), ("threshold hits~10%", -0.1, 0.1), ("threshold hits~50%", -0.5, 0.5),
                         ("threshold hits=100%", -2.0, 2.0)):
        run(name, lambda lo=lo, hi=hi: nat.select_threshold(attr, None, lo, hi, data, mask, edited, 3, counts=cnt), 4 * n)
    noise = torch.rand((N, N), device=dev, generator=g)
    run("threshold noise hits=20%", lambda: nat.select_threshold(noise, None, 0.0, 0.2, data, mask, edited, 3, counts=cnt), 4 * n)
    del noise

    m2 = (torch.rand((N, N), device=dev, generator=g) < 0.3).to(torch.uint8)
    out = torch.zeros((N, N), dtype=torch.uint8, device=dev)
    run("mask_op union", lambda: nat.layer_op("union", None, mask, None, m2, None, out), 3 * n)
    d2 = torch.zeros((N, N), dtype=torch.uint8, device=dev)
    dout = torch.zeros((N, N), dtype=torch.uint8, device=dev)
    run("layer_op union u8", lambda: nat.layer_op("union", data, mask, d2, m2, dout, out), 6 * n)
    if not want or any(w in "layer chain" for w in want):
        ops = ["union", "union", "intersection", "difference", "union", "masking", "difference", "union"]   # ops[0] is ignored
        for label, p in (("sparse (5%% blobs)", 0.05), ("dense (60%% blobs)", 0.6)):
            cm = []
            for k in range(8):          # coherent blobs: threshold a smooth field
                yy, xx = torch.meshgrid(torch.linspace(0, 9 + k, N, device=dev), torch.linspace(0, 7 + k, N, device=dev), indexing="ij")
                f = torch.sin(xx + k) * torch.cos(yy - k)
                thr_v = torch.quantile(f[::64, ::64].flatten(), 1.0 - p)
                cm.append((f > thr_v).to(torch.uint8))
                del yy, xx, f
            cd = [torch.full((N, N), k + 1, dtype=torch.uint8, device=dev) for k in range(8)]
            run("layer chain 2 (layer_op union u8) " + label % (), lambda: nat.layer_op("union", cd[0], cm[0], cd[1], cm[1], dout, out), 6 * n)
            run("layer chain 8 u8 " + label % (), lambda: nat.layer_chain(cd, cm, ops, dout, out), 18 * n)
            run("layer chain 8 u8 eager " + label % (), lambda: nat.layer_chain(cd, cm, ops, dout, out, lazy=False), 18 * n)
            cd32 = [torch.full((N, N), k + 1, dtype=torch.int32, device=dev) for k in range(4)]
            d32 = torch.zeros((N, N), dtype=torch.int32, device=dev)
            run("layer chain 4 i32 " + label % (), lambda: nat.layer_chain(cd32, cm[:4], ops[:4], d32, out), 25 * n)
            run("layer chain 4 i32 eager " + label % (), lambda: nat.layer_chain(cd32, cm[:4], ops[:4], d32, out, lazy=False), 25 * n)
            del cm, cd, cd32, d32
    run("memset 1 plane (torch)", lambda: out.zero_(), n)
    run("copy 1 plane (torch)", lambda: out.copy_(m2), 2 * n)

    cov = torch.zeros((N, N), dtype=torch.uint8, device=dev)
    cov[N // 100: N - N // 100, N // 100: N - N // 100] = 1
    run("outline_mask r=1", lambda: nat.outline_mask(cov, 1), 2 * n)
    ring = nat.outline_mask(cov, 1)
    edited.zero_()
    edited[N // 2 - 500: N // 2 + 500, N // 2 - 500: N // 2 + 500] = 1
    run("padding r=1 (interior stroke)", lambda: nat.apply_padding(ring, edited, 1, data, mask, 3, counts=cnt), n)
    edited[: N // 50, :] = 1
    run("padding r=1 (stroke on border)", lambda: nat.apply_padding(ring, edited, 1, data, mask, 3, counts=cnt), n)
    zero_ring = torch.zeros_like(ring)
    run("padding r=1 (empty outline)", lambda: nat.apply_padding(zero_ring, edited, 1, data, mask, 3, counts=cnt), n)
    rows_only = torch.zeros_like(ring)
    rows_only[N // 100 - 1, :] = 1
    run("padding r=1 (one outline row)", lambda: nat.apply_padding(rows_only, edited, 1, data, mask, 3, counts=cnt), n)
    del cov, ring, zero_ring, rows_only

    pos = torch.rand((3, N, N), device=dev, generator=g)
    run("sphere few hits", lambda: nat.select_sphere(pos, (0.5, 0.5, 0.5), 0.05, data, mask, edited, 3, counts=cnt), 12 * n)
    run("sphere 50% hits", lambda: nat.select_sphere(pos, (0.5, 0.5, 0.5), 0.62, data, mask, edited, 3, counts=cnt), 12 * n)
    if not want or any(w in "display pack" for w in want):
        from paper_2501_14807_b200.display import Palette
        pal = Palette.grayscale()
        pos_pts, col_pts = np.asarray(pal.positions, dtype=np.float64), np.asarray(pal.colours, dtype=np.float64)
        rgba = torch.empty((N, N, 4), dtype=torch.uint8, device=dev)
        dd = torch.randint(0, 256, (N, N), device=dev, generator=g, dtype=torch.int32).to(torch.uint8)
        half = (torch.rand((N, N), device=dev, generator=g) < 0.5).to(torch.uint8)
        full = torch.ones((N, N), dtype=torch.uint8, device=dev)
        run("display u8 (all valid)", lambda: nat.resolve_display(dd, full, 0.0, 255.0, pos_pts, col_pts, out=rgba), 6 * n)
        run("display u8 (50% noise mask)", lambda: nat.resolve_display(dd, half, 0.0, 255.0, pos_pts, col_pts, out=rgba), 6 * n)
        df = torch.rand((N, N), device=dev, generator=g)
        run("display f32 (all valid)", lambda: nat.resolve_display(df, full, 0.0, 1.0, pos_pts, col_pts, out=rgba), 9 * n)
        bits = nat.pack_mask(half)
        run("pack_mask", lambda: nat.pack_mask(half), n + n // 8)
        outm = torch.empty((N, N), dtype=torch.uint8, device=dev)
        run("unpack_mask", lambda: nat.unpack_mask(bits, N * N, outm), n + n // 8)
        del rgba, dd, half, full, df, bits
    # smooth "surface" positions (a heightfield over the atlas) for the footprint-culled brushes
    if not want or any(w in "sphere culled" for w in want):
        yy, xx = torch.meshgrid(torch.linspace(0, 1, N, device=dev), torch.linspace(0, 1, N, device=dev), indexing="ij")
        spos = torch.stack([xx, yy, 0.1 * torch.sin(7 * xx) * torch.cos(5 * yy)]).contiguous()
        del yy, xx
        tiles = nat.tile_boxes(spos)
        for r in (0.005, 0.02, 0.08, 0.3):
            run("sphere stream  r=%.3f" % r, lambda r=r: nat.select_sphere(spos, (0.5, 0.5, 0.0), r, data, mask, edited, 3, counts=cnt), 12 * n)
            run("sphere culled  r=%.3f" % r, lambda r=r: nat.select_sphere(spos, (0.5, 0.5, 0.0), r, data, mask, edited, 3, counts=cnt, tiles=tiles), 12 * n)
        del spos, tiles
    area = pos[0]
    masks = [m2, mask, out, d2]
    run("area L=1", lambda: nat.layer_area(area, masks[:1], sums=torch.zeros(1, dtype=torch.float64, device=dev),
                                           counts=torch.zeros(1, dtype=torch.int64, device=dev)), 5 * n)
    run("area L=4 (noise+coherent)", lambda: nat.layer_area(area, masks, sums=torch.zeros(4, dtype=torch.float64, device=dev),
                                                            counts=torch.zeros(4, dtype=torch.int64, device=dev)), 8 * n)


if __name__ == "__main__":
    main()
