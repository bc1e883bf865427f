import sys, time, cProfile, pstats, io
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import paper_2501_14807_b200 as ml
from paper_2501_14807_b200 import synth, _native as nat
mesh = synth.heightfield_mesh(707, margin=0.01)
A = 16384
cam = synth.default_camera(1024, 1024, eye=(.5, .5, 1.6), target=(.5, .5, 0), fovy=40, near=.2, far=5)
surf = ml.build_surface_map(mesh, A, A)
ctx = ml.StrokeContext(mesh, cam, ml.render_depth(mesh, cam), surf)
pool = ml.TexturePool(budget_texels=2**34)
layer = ml.create_layer("a", "uint8", A, A, pool=pool)
shape = nat._as_dev_bytes(synth.circle_shape(70), "cuda")
rng = np.random.default_rng(0)
tools = [ml.EditingTool(px=float(rng.uniform(300, 700)), py=float(rng.uniform(300, 700)), shape=shape, value=7) for _ in range(200)]
for t in tools[:5]: ml.apply_stroke(ctx, t, layer)
torch.cuda.synchronize()
for cull in (True, False):
    t0 = time.perf_counter()
    for t in tools: ml.apply_stroke(ctx, t, layer, cull=cull)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print("cull=%s: host issue %.1f us/stroke, total %.1f us/stroke" % (cull, (t1 - t0) / 200 * 1e6, (t2 - t0) / 200 * 1e6))
pr = cProfile.Profile(); pr.enable()
for t in tools: ml.apply_stroke(ctx, t, layer)
pr.disable(); torch.cuda.synchronize()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(18); print(s.getvalue()[:3500])
