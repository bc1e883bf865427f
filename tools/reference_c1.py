#!/usr/bin/env python
"""Time the REFERENCE's own numpy kernels on BASELINE config C1 (icosphere level 5 = 20,480 triangles,
1024^2 atlas, 512^2 window, one r = 40 px stroke) next to the oracle's C restatement, and check that both
give the same planes.  Runs only where /root/reference exists (the build container, not the GPU box):

    python tools/reference_c1.py > profiles/r1_reference_c1.json

The CUDA numbers for the same case are in profiles/r1_config_times.json (tools/config_times.py)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")
from meshlayers import _kernels_numpy as KN  # noqa: E402  (the reference itself)
import helpers  # noqa: E402
from oracle import kn  # noqa: E402


def timed(fn):
    t0 = time.perf_counter()
    r = fn()
    return r, time.perf_counter() - t0


def main():
    A, W = 1024, 512
    s = helpers.tea_scene_inputs(5, A, W, 40, (W / 2.0, W / 2.0))
    out = {"config": "C1: icosphere level 5 (%d triangles), %dx%d atlas, %dx%d window, circular tool r = 40 px"
                     % (s["mesh"].num_triangles, A, A, W, W),
           "host": "build container CPU (%d cores visible); the GPU box's host differs" % os.cpu_count()}
    cov_r, cov_c = np.zeros((A, A), np.uint8), np.zeros((A, A), np.uint8)
    n_r, t_r = timed(lambda: KN.coverage_fill(s["tri_xy"], A, A, cov_r))
    n_c, t_c = timed(lambda: kn.coverage_fill(s["tri_xy"], A, A, cov_c))
    assert n_r == n_c and np.array_equal(cov_r, cov_c)
    out["coverage_fill"] = {"reference_numpy_s": t_r, "c_port_1_thread_s": t_c, "covered": int(n_r)}
    d_r, d_c = np.ones((W, W), np.float32), np.ones((W, W), np.float32)
    _, t_r = timed(lambda: KN.raster_depth(s["win_xy"], s["win_zn"], d_r))
    _, t_c = timed(lambda: kn.raster_depth(s["win_xy"], s["win_zn"], d_c))
    assert np.array_equal(d_r.view(np.uint32), d_c.view(np.uint32))
    out["raster_depth"] = {"reference_numpy_s": t_r, "c_port_1_thread_s": t_c}
    planes = [[np.zeros((A, A), np.uint8), np.zeros((A, A), bool), np.zeros((A, A), bool)] for _ in range(3)]
    args = (s["tri_xy"], s["tri_clip"], float(W), float(W), d_r, 1e-4, s["sfx"], s["sfy"], s["bx"], s["by"], s["shape"])
    r_r, t_r = timed(lambda: KN.raster_tea(*args, *planes[0], 7))
    r_c, t_c = timed(lambda: kn.raster_tea(*args, *planes[1], 7))
    r_m, t_m = timed(lambda: kn.raster_tea(*args, *planes[2], 7, threads=0))
    assert tuple(r_r) == tuple(r_c) == tuple(r_m)
    for a, b, c in zip(*planes):
        assert np.array_equal(a, b) and np.array_equal(a, c)
    out["raster_tea"] = {"reference_numpy_s": t_r, "c_port_1_thread_s": t_c, "c_port_all_threads_s": t_m,
                         "threads": kn.max_threads(), "edited": int(r_r[0]), "fragments": int(r_r[1])}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
