#!/usr/bin/env python
"""Device time per stroke (apply_stroke = TEA, stroke = TEA + TPA through ml_stroke) at 16384^2 with the
1M-triangle mesh for tool radii 10 / 70 / 200 px: 50 strokes back to back between two CUDA events.
Tuning aid; the paper-style sweep with the SPEC's CSV is `python -m paper_2501_14807_b200.bench`."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2501_14807_b200 as ml
from paper_2501_14807_b200 import synth, _native as nat
mesh = synth.heightfield_mesh(707, margin=0.01)
A = 16384
cam = synth.default_camera(1024, 1024, eye=(.5, .5, 1.6), target=(.5, .5, 0), fovy=40, near=.2, far=5)
surf = ml.build_surface_map(mesh, A, A)
ctx = ml.StrokeContext(mesh, cam, ml.render_depth(mesh, cam), surf)
outline = ml.build_outline_mask(surf.coverage, thickness=1)
pool = ml.TexturePool(budget_texels=2**34)
layer = ml.create_layer("a", "uint8", A, A, pool=pool)
for rad in (10, 70, 200):
    shape = nat._as_dev_bytes(synth.circle_shape(rad), "cuda")
    rng = np.random.default_rng(0)
    tools = [ml.EditingTool(px=float(rng.uniform(300, 700)), py=float(rng.uniform(300, 700)), shape=shape, value=7) for _ in range(60)]
    for name, fn in (("apply_stroke", lambda t: ml.apply_stroke(ctx, t, layer)), ("stroke", lambda t: ml.stroke(ctx, t, layer, outline))):
        for t in tools[:10]: fn(t)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for t in tools[10:]: r = fn(t)
        b.record(); torch.cuda.synchronize()
        print("r=%3d %-13s %.1f us/stroke  (edited %d)" % (rad, name, a.elapsed_time(b) / 50 * 1e3, r.edited_count), flush=True)
