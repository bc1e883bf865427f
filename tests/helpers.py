"""Shared scene builders for tests (and tests/golden/make_golden.py)."""
import glob
import os

import numpy as np

from paper_2501_14807_b200 import synth
from paper_2501_14807_b200.mesh_core import window_triangles

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def golden_names(prefix):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


def tea_scene_inputs(level, atlas, window, tool_r, tool_xy):
    """Icosphere + chart-grid atlas + default camera + circular tool; everything except the depth
    plane (which the fixture stores, because the reference rendered it)."""
    mesh = synth.icosphere_mesh(int(level))
    cam = synth.default_camera(int(window), int(window))
    win_xy, win_zn = window_triangles(mesh, cam)
    tri_xy = mesh.tri_uv_texels(int(atlas), int(atlas))
    clip = cam.clip_coords(mesh.vertices)[mesh.triangles]
    shape = synth.circle_shape(int(tool_r))
    tw = th = shape.shape[0]
    sfx, sfy = window / (2.0 * tw), window / (2.0 * th)
    bx = 0.5 - (float(tool_xy[0]) - 0.5 * window) / tw
    by = 0.5 - (float(tool_xy[1]) - 0.5 * window) / th
    return dict(mesh=mesh, cam=cam, win_xy=win_xy, win_zn=win_zn, tri_xy=tri_xy, tri_clip=clip,
                shape=shape, sfx=float(sfx), sfy=float(sfy), bx=float(bx), by=float(by))


def eps_of(fix):
    """Fixture eps with the Python type the reference was called with (float vs np.float64)."""
    return np.float64(fix["eps"]) if bool(fix["eps_is_np64"]) else float(fix["eps"])


def random_tea_case(seed, ntri=200, w=64, h=64, plane_dtype=np.uint8, value=7, tri_dtype=np.float64,
                    eps=1e-4):
    """Random TEA stroke inputs (same recipe as the tea_rand_* fixtures)."""
    rng = np.random.default_rng(seed)
    tri = synth.random_soup(rng, ntri, float(max(w, h)), dtype=np.float64)
    tri[..., 1] *= h / float(max(w, h))
    tri = tri.astype(tri_dtype)
    ww, wh = 37.0, 29.0
    clip = np.empty((ntri, 3, 4))
    wc = rng.uniform(0.5, 3.0, size=(ntri, 3))
    wc[rng.random((ntri, 3)) < 0.08] *= -1.0
    clip[..., 3] = wc
    clip[..., 0] = rng.uniform(-1.4, 1.4, size=(ntri, 3)) * np.abs(wc)
    clip[..., 1] = rng.uniform(-1.4, 1.4, size=(ntri, 3)) * np.abs(wc)
    clip[..., 2] = rng.uniform(-1.0, 1.0, size=(ntri, 3)) * np.abs(wc)
    clip = clip.astype(tri_dtype)
    depth = rng.uniform(0.2, 1.0, size=(int(wh), int(ww))).astype(np.float32)
    shape = (rng.random((9, 11)) < 0.7).astype(np.uint8)
    data = rng.integers(0, 5, size=(h, w)).astype(plane_dtype)
    mask = rng.random((h, w)) < 0.1
    edited = (rng.random((h, w)) < 0.05).astype(np.uint8)
    return dict(tri_xy=tri, tri_clip=clip, ww=ww, wh=wh, depth=depth, eps=eps, sfx=1.3, sfy=0.9,
                bx=0.45, by=0.55, shape=shape, data=data, mask=mask, edited=edited, value=value)


def tea_args(c):
    return (c["tri_xy"], c["tri_clip"], c["ww"], c["wh"], c["depth"], c["eps"], c["sfx"], c["sfy"],
            c["bx"], c["by"], c["shape"])
