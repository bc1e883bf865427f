"""Generate tests/golden/*.npz by running the REFERENCE's own numpy kernels.

Run in the build container only (needs /root/reference, which does not exist on the GPU box):

    python tests/golden/make_golden.py

Each fixture stores the seeded inputs and the planes / counts the reference produced, so the
oracle (oracle/kn_port.c) and the CUDA library can be pinned against the reference without the
reference being present.  Scenes deliberately mix float32 / float64 inputs, both windings,
vertices snapped onto texel centres and corners (tie rule), degenerate triangles, pre-dirtied
planes, all plane kinds and both eps promotion modes.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from meshlayers import _kernels_numpy as KN  # noqa: E402  (the reference itself)

from paper_2501_14807_b200 import synth  # noqa: E402
sys.path.insert(0, os.path.dirname(HERE))
import helpers  # noqa: E402  (tests/helpers.py)


def soup(rng, ntri, w, h, dtype):
    tri = synth.random_soup(rng, ntri, float(max(w, h)), dtype=np.float64)
    tri[..., 1] *= h / float(max(w, h))
    return tri.astype(dtype)


def gen_coverage(seed, ntri, w, h, dtype, dirty):
    rng = np.random.default_rng(seed)
    tri = soup(rng, ntri, w, h, dtype)
    out0 = np.zeros((h, w), np.uint8)
    if dirty:
        out0[rng.random((h, w)) < 0.05] = 1
        out0[rng.random((h, w)) < 0.02] = 7          # non-{0,1} bytes must become exactly 1
    out = out0.copy()
    written = KN.coverage_fill(tri, w, h, out)
    return dict(tri_xy=tri, width=w, height=h, out0=out0, out=out, written=written)


def gen_depth(seed, ntri, w, h, dtype):
    rng = np.random.default_rng(seed)
    tri = soup(rng, ntri, w, h, dtype)
    zn = rng.uniform(-1.3, 1.1, size=(ntri, 3)).astype(dtype)
    d0 = np.ones((h, w), np.float32)
    d0[rng.random((h, w)) < 0.1] = np.float32(0.4)
    depth = d0.copy()
    KN.raster_depth(tri, zn, depth)                  # count is order dependent: not stored
    return dict(tri_xy=tri, tri_zn=zn, depth0=d0, depth=depth)


def gen_tea_random(seed, ntri, w, h, dtype, plane_dtype, eps, value):
    rng = np.random.default_rng(seed)
    tri = soup(rng, ntri, w, h, dtype)
    ww, wh = 37.0, 29.0
    clip = np.empty((ntri, 3, 4))
    wc = rng.uniform(0.5, 3.0, size=(ntri, 3))
    wc[rng.random((ntri, 3)) < 0.08] *= -1.0         # some vertices behind the projector
    clip[..., 3] = wc
    clip[..., 0] = rng.uniform(-1.4, 1.4, size=(ntri, 3)) * np.abs(wc)
    clip[..., 1] = rng.uniform(-1.4, 1.4, size=(ntri, 3)) * np.abs(wc)
    clip[..., 2] = rng.uniform(-1.0, 1.0, size=(ntri, 3)) * np.abs(wc)
    clip = clip.astype(dtype)
    depth = rng.uniform(0.2, 1.0, size=(int(wh), int(ww))).astype(np.float32)
    th, tw = 9, 11
    shape = (rng.random((th, tw)) < 0.7).astype(np.uint8)
    sfx, sfy, bx, by = 1.3, 0.9, 0.45, 0.55
    data0 = (rng.integers(0, 5, size=(h, w))).astype(plane_dtype)
    mask0 = (rng.random((h, w)) < 0.1)
    edited0 = (rng.random((h, w)) < 0.05).astype(np.uint8)
    data, mask, edited = data0.copy(), mask0.copy(), edited0.copy()
    ec, fr = KN.raster_tea(tri, clip, ww, wh, depth, eps, sfx, sfy, bx, by, shape, data, mask, edited, value)
    return dict(tri_xy=tri, tri_clip=clip, ww=ww, wh=wh, depth=depth, eps=np.float64(eps),
                eps_is_np64=isinstance(eps, np.float64), sfx=sfx, sfy=sfy, bx=bx, by=by, shape=shape,
                data0=data0, mask0=mask0, edited0=edited0, data=data, mask=mask, edited=edited,
                value=np.array(value, dtype=plane_dtype), edited_count=ec, fragments=fr)


def gen_tea_scene(level, atlas, window, tool_r, tool_xy, eps):
    """Icosphere + chart-grid atlas + perspective camera + circular tool (small)."""
    s = helpers.tea_scene_inputs(level, atlas, window, tool_r, tool_xy)
    depth = np.ones((window, window), np.float32)
    KN.raster_depth(s["win_xy"], s["win_zn"], depth)
    data = np.zeros((atlas, atlas), np.uint8)
    mask = np.zeros((atlas, atlas), bool)
    edited = np.zeros((atlas, atlas), bool)
    ec, fr = KN.raster_tea(s["tri_xy"], s["tri_clip"], float(window), float(window), depth, eps,
                           s["sfx"], s["sfy"], s["bx"], s["by"], s["shape"], data, mask, edited, 7)
    return dict(level=level, atlas=atlas, window=window, tool_r=tool_r, tool_xy=np.array(tool_xy, float),
                eps=np.float64(eps), eps_is_np64=False, depth=depth, data=np.packbits(data != 0),
                data_value=7, mask=np.packbits(mask), edited=np.packbits(edited),
                edited_count=ec, fragments=fr,
                cov_count=int(_coverage_count(s["tri_xy"], atlas)))


def _coverage_count(tri_xy, atlas):
    out = np.zeros((atlas, atlas), np.uint8)
    return KN.coverage_fill(tri_xy, atlas, atlas, out)


def main():
    out = {}
    out["coverage_a"] = gen_coverage(11, 160, 48, 40, np.float64, dirty=False)
    out["coverage_b"] = gen_coverage(12, 160, 33, 57, np.float32, dirty=True)
    out["coverage_big"] = gen_coverage(13, 12, 96, 96, np.float64, dirty=False)
    out["depth_a"] = gen_depth(21, 140, 40, 36, np.float64)
    out["depth_b"] = gen_depth(22, 140, 31, 45, np.float32)
    kinds = [(np.uint8, 7), (np.int16, -1234), (np.float32, 2.5), (np.uint32, 4000000000),
             (np.float16, 0.333), (np.int8, -3), (np.int32, -70000)]
    for k, (dt, val) in enumerate(kinds):
        eps = 1e-4 if k % 2 == 0 else np.float64(1e-4)
        out["tea_rand_%d" % k] = gen_tea_random(31 + k, 150, 44, 38, np.float64 if k % 3 else np.float32,
                                                dt, eps, val)
    out["tea_scene_centre"] = gen_tea_scene(2, 128, 96, 12, (48.0, 48.0), 1e-4)
    out["tea_scene_edge"] = gen_tea_scene(2, 128, 96, 20, (80.0, 30.0), 1e-4)
    out["tea_scene_background"] = gen_tea_scene(1, 64, 64, 4, (3.0, 3.0), 1e-4)
    # eps promotion (KN:185): Python-float eps is added in float32, np.float64 eps in float64
    tri = np.array([[[-10.0, -10.0], [30.0, -10.0], [-10.0, 30.0]]])
    dv, eps = np.float32(0.6), 1e-9
    clip = np.zeros((1, 3, 4))
    clip[..., 3] = 1.0
    clip[..., 2] = (float(dv) + 0.5 * eps) * 2.0 - 1.0
    counts = []
    for e in (eps, np.float64(eps)):
        data, mask, edited = np.zeros((4, 4), np.uint8), np.zeros((4, 4), bool), np.zeros((4, 4), bool)
        counts.append(KN.raster_tea(tri, clip, 4.0, 4.0, np.full((4, 4), dv, np.float32), e, 0.5, 0.5, 0.5,
                                    0.5, np.ones((1, 1), np.uint8), data, mask, edited, 1)[0])
    out["epsmode"] = dict(tri_xy=tri, tri_clip=clip, depth_value=dv, eps=np.float64(eps),
                          edited_weak=counts[0], edited_f64=counts[1])
    for name, d in out.items():
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)
        print(name, {k: (v.shape if hasattr(v, "shape") and getattr(v, "ndim", 0) else v) for k, v in d.items()
                     if k in ("written", "edited_count", "fragments", "cov_count")})


if __name__ == "__main__":
    main()
