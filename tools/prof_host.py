#!/usr/bin/env python
"""Host-side issue cost of the per-stroke public API calls (how long Python + ctypes take to queue
a stroke) next to the total time per stroke; cProfile of the hottest call.  Tuning aid."""
import cProfile
import io
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_14807_b200 as ml  # noqa: E402
from paper_2501_14807_b200 import synth, _native as nat  # noqa: E402

mesh = synth.heightfield_mesh(707, margin=0.01)
A = 16384
cam = synth.default_camera(1024, 1024, eye=(.5, .5, 1.6), target=(.5, .5, 0), fovy=40, near=.2, far=5)
surf = ml.build_surface_map(mesh, A, A)
ctx = ml.StrokeContext(mesh, cam, ml.render_depth(mesh, cam), surf)
outline = ml.build_outline_mask(surf.coverage, thickness=1)
pool = ml.TexturePool(budget_texels=2**34)
layer = ml.create_layer("a", "uint8", A, A, pool=pool)
edited = torch.zeros((A, A), dtype=torch.uint8, device="cuda")
shape = nat._as_dev_bytes(synth.circle_shape(70), "cuda")
rng = np.random.default_rng(0)
N = 200
tools = [ml.EditingTool(px=float(rng.uniform(300, 700)), py=float(rng.uniform(300, 700)), shape=shape, value=7) for _ in range(N)]
strokes, labels = synth.sphere_strokes(mesh, N, seed=5, rmin_frac=0.01, rmax_frac=0.05)


def timed(name, fn):
    for i in range(5):
        fn(i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(N):
        fn(i)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print("%-28s host issue %6.1f us/call, total %6.1f us/call" % (name, (t1 - t0) / N * 1e6, (t2 - t0) / N * 1e6), flush=True)


for cull in (True, False):
    timed("apply_stroke cull=%s" % cull, lambda i: ml.apply_stroke(ctx, tools[i], layer, cull=cull))
    timed("stroke (TEA+TPA) cull=%s" % cull, lambda i: ml.stroke(ctx, tools[i], layer, outline, cull=cull))
    timed("select_sphere cull=%s" % cull, lambda i: ml.select_sphere(surf, layer, strokes[i, :3], strokes[i, 3], int(labels[i]),
                                                                   edited=edited, cull=cull))
which = sys.argv[1] if len(sys.argv) > 1 else "sphere"
pr = cProfile.Profile()
pr.enable()
for i in range(N):
    if which == "sphere":
        ml.select_sphere(surf, layer, strokes[i, :3], strokes[i, 3], int(labels[i]), edited=edited)
    else:
        ml.stroke(ctx, tools[i], layer, outline)
pr.disable()
torch.cuda.synchronize()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(22)
print(s.getvalue()[:4500])
