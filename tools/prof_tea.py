#!/usr/bin/env python
"""A few culled TEA strokes with a given tool radius at 16384^2 (ncu target for tea_eval_kernel) + device time.

    python tools/prof_tea.py [radius_px=200] [reps=5]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import argparse
    import numpy as np
    import torch
    import paper_2501_14807_b200 as ml
    from paper_2501_14807_b200 import synth
    import bench as B
    r = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    wl = B.Workload(argparse.Namespace(atlas=16384, layers=8, quads=707, window=1024), 1)
    surf = ml.build_surface_map(wl.mesh, 16384, 16384)
    depth = ml.render_depth(wl.mesh, wl.cam)
    ctx = ml.StrokeContext(wl.mesh, wl.cam, depth, surf)
    layer = ml.create_layer("L", "uint8", 16384, 16384, pool=ml.TexturePool(budget_texels=2 ** 33))
    shape = torch.from_numpy(synth.circle_shape(r)).cuda()
    ts, cnt = [], None
    for k in range(reps + 1):
        tool = ml.EditingTool(px=512.0 + 3 * k, py=500.0, shape=shape, value=7)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        res = ml.apply_stroke(ctx, tool, layer, eps=wl.eps)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        cnt = res.edited_count
    print("radius %d px: %.3f ms per culled TEA stroke (median of %d), %d texels edited" % (r, float(np.median(ts[1:])), reps, cnt))


if __name__ == "__main__":
    main()
