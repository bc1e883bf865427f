"""CPU-only tests of the host side: error surface, projection formulas, C-ABI symbols, and the
"fails loudly without CUDA" contract.  No compute calls are made without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2501_14807_b200 as ml
from paper_2501_14807_b200 import _native, errors, sharding, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ------------------------------------------------------------------ errors (reference errors.py:4-97)

REFERENCE_CODES = {
    "MeshLayersError": "error", "ParseError": "parse_error", "UVRangeError": "uv_range",
    "MissingUVs": "missing_uvs", "EmptyMesh": "empty_mesh", "DegenerateCamera": "degenerate_camera",
    "CapacityExceeded": "capacity_exceeded", "TargetMismatch": "target_mismatch", "BadPalette": "bad_palette",
    "UnknownTable": "unknown_table", "BadMagic": "bad_magic", "UnsupportedVersion": "unsupported_version",
    "TruncatedStream": "truncated_stream", "ChecksumMismatch": "checksum_mismatch", "StaleDepth": "stale_depth",
    "LayerMeshMismatch": "layer_mesh_mismatch", "MemoryBudgetExceeded": "memory_budget_exceeded",
    "DuplicateTable": "duplicate_table", "BadSchema": "bad_schema", "SchemaViolation": "schema_violation",
    "ReservedKey": "reserved_key", "UnknownLayer": "unknown_layer", "BindFailure": "bind_failure",
    "BadRequest": "bad_request",
}


def test_error_classes_and_wire_codes():
    for name, code in REFERENCE_CODES.items():
        cls = getattr(errors, name)
        assert cls.code == code and issubclass(cls, errors.MeshLayersError)
        assert getattr(ml, name) is cls
    assert issubclass(errors.UVRangeError, errors.ParseError)          # errors.py:12
    assert issubclass(errors.MeshLayersError, Exception)
    with pytest.raises(errors.MeshLayersError):
        raise errors.StaleDepth("x")


# ------------------------------------------------------------------ C ABI

def _header_symbols():
    with open(os.path.join(ROOT, "include", "meshlayers_b200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(ml_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib_path = _native.LIB_PATH
    assert os.path.exists(lib_path), "run `python -m paper_2501_14807_b200.build` (driver build() does)"
    L = ctypes.CDLL(lib_path)
    declared = _header_symbols()
    assert len(declared) >= 24
    for sym in declared:
        assert hasattr(L, sym), sym
    assert set(declared) == set(_native.EXPORTED_SYMBOLS)
    assert _native.lib().ml_version() >= 100
    assert int(_native.lib().ml_raster_workspace_bytes(1000)) >= 1000 * 12


def test_no_cpu_fallback_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present: the loud-failure path is not reachable")
    with pytest.raises(errors.BackendUnavailable):
        _native.require_cuda()
    mesh = synth.icosphere_mesh(1)
    with pytest.raises(errors.BackendUnavailable):
        ml.build_surface_map(mesh, 32, 32)
    with pytest.raises(errors.BackendUnavailable):
        ml.uv_coverage(mesh, 32)
    with pytest.raises(errors.BackendUnavailable):
        ml.TexturePool().acquire(8, 8, "uint8")
    # the numpy (host-buffer) entry point goes straight to the CUDA library and reports no device
    with pytest.raises(errors.MeshLayersError):
        _native.coverage_fill(np.zeros((1, 3, 2)) + [[0, 0], [4, 0], [0, 4]], 8, 8, np.zeros((8, 8), np.uint8))


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2501_14807_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert not re.search(r"^\s*(from|import)\s+oracle\b", src, re.M), fn


# ------------------------------------------------------------------ projection formulas

def _cam(w, h):
    return synth.default_camera(w, h)


def test_tool_projection_known_answers():
    shape = np.ones((100, 100), np.uint8)
    p = ml.compute_tool_projection(_cam(800, 600), ml.EditingTool(400, 300, shape))
    assert p.scale == (4.0, 3.0) and p.translate == (0.0, 0.0)
    p = ml.compute_tool_projection(_cam(1024, 1024), ml.EditingTool(512, 512, np.ones((256, 256), np.uint8)))
    assert p.scale == (2.0, 2.0) and p.translate == (0.0, 0.0)
    p = ml.compute_tool_projection(_cam(800, 600), ml.EditingTool(0, 0, shape))
    assert p.translate == (-4.0, -3.0)
    assert p.kernel_factors == (4.0, 3.0, 4.5, 3.5)


def test_tool_projection_random_tuples():
    rng = np.random.default_rng(0)
    for _ in range(100):
        ww, wh = int(rng.integers(1, 4000)), int(rng.integers(1, 4000))
        tw, th = int(rng.integers(1, 500)), int(rng.integers(1, 500))
        px, py = rng.uniform(0, ww), rng.uniform(0, wh)
        p = ml.compute_tool_projection(_cam(ww, wh), ml.EditingTool(px, py, np.ones((th, tw), np.uint8)))
        want = (ww / (2 * tw), wh / (2 * th), (px - 0.5 * ww) / tw, (py - 0.5 * wh) / th)
        got = p.scale + p.translate
        assert all(abs(g - w) <= 1e-12 * max(1.0, abs(w)) for g, w in zip(got, want))
        # centre of the tool maps to s = t = 0.5 through the kernel's tool map
        sfx, sfy, bx, by = p.kernel_factors
        xn, yn = 2 * px / ww - 1, 2 * py / wh - 1
        assert abs(sfx * xn + bx - 0.5) < 1e-9 and abs(sfy * yn + by - 0.5) < 1e-9


def test_project_fragment():
    assert ml.project_fragment(0.5, 0.5, 1.0) == (0.5, 0.5)
    assert ml.project_fragment(2.0, 2.0, 4.0) == (0.5, 0.5)
    assert ml.project_fragment(1.5, 0.5, 1.0) is None
    assert ml.project_fragment(0.5, 0.5, 0.0) is None and ml.project_fragment(0.5, 0.5, -1.0) is None
    assert ml.project_fragment(1.0, 0.0, 1.0) == (1.0, 0.0)                    # closed interval, KN:189


def test_degenerate_camera_and_mesh_validation():
    with pytest.raises(errors.DegenerateCamera):
        ml.Camera(view=np.eye(4), projection=np.zeros((4, 4)), width=10, height=10)
    with pytest.raises(errors.DegenerateCamera):
        ml.Camera(view=np.eye(4), projection=np.eye(4), width=0, height=10)
    with pytest.raises(errors.UVRangeError):
        ml.TriangleMesh(np.zeros((3, 3)), np.zeros((3, 3)), np.array([[0, 0], [2, 0], [0, 1.0]]), np.array([[0, 1, 2]]))
    with pytest.raises(errors.MissingUVs):
        ml.TriangleMesh(np.zeros((3, 3)), np.zeros((3, 3)), None, np.array([[0, 1, 2]]))


def test_camera_generation_follows_every_change():
    cam = synth.default_camera(64, 48)
    k0, g0 = cam.state_key(), cam.generation
    cam.set_view(synth.look_at((1.0, 2.0, 3.0), (0.0, 0.0, 0.0)))
    assert cam.generation == g0 + 1 and cam.state_key() != k0
    cam.projection = synth.perspective(30.0, 64 / 48, 0.1, 9.0)
    cam.width = 32
    assert cam.generation == g0 + 3
    with pytest.raises(ml.DegenerateCamera):
        cam.set_projection(np.zeros((4, 4)))
    assert cam.generation == g0 + 3 and np.linalg.det(cam.projection) != 0.0          # a rejected change leaves no trace
    k1 = cam.state_key()
    cam.view[1, 3] += 1.0                                                             # in-place edit: same generation,
    assert cam.generation == g0 + 3 and cam.state_key() != k1                         # different key


def test_triangles_crossing_the_eye_plane_still_occlude():                       # SPEC occlusion safety
    """A triangle with a vertex BEHIND the camera is clipped to w >= eps_w for the depth pass instead of being
    dropped: its visible part must hide the wall behind it.  (Oracle depth pass; host preparation only.)"""
    from oracle import kn
    from paper_2501_14807_b200.mesh_core import TriangleMesh, window_triangles, _clip_eye_plane
    cam = synth.default_camera(64, 64, eye=(0.0, 0.0, 0.0), target=(0.0, 0.0, -1.0), fovy=60.0, near=0.1, far=10.0)
    wall = np.array([[-4, -4, -3], [4, -4, -3], [4, 4, -3], [-4, 4, -3]], float)
    blade = np.array([[-3, -3, -2], [3, -3, -2], [0, 4, 1]], float)               # third vertex behind the eye
    verts = np.concatenate([wall, blade])
    tris = np.array([[0, 1, 2], [0, 2, 3], [4, 5, 6]])
    mesh = TriangleMesh(vertices=verts, normals=None, uvs=np.zeros((7, 2)), triangles=tris)
    xy, zn = window_triangles(mesh, cam)
    assert xy.shape[0] == 2 + 2 and np.isfinite(xy).all() and np.isfinite(zn).all()   # blade: two inside vertices -> 2 triangles
    depth = np.ones((64, 64), np.float32)
    kn.raster_depth(xy, zn, depth)
    only_wall = np.ones((64, 64), np.float32)
    kn.raster_depth(xy[:2], zn[:2], only_wall)
    assert depth[20, 32] < only_wall[20, 32] < 1.0                                   # the blade is nearer than the wall there
    assert (depth <= only_wall).all()
    # clipping keeps the winding and stays on the visible side
    clip = cam.clip_coords(mesh.vertices)[mesh.triangles][2:3]
    parts = _clip_eye_plane(clip, 1e-9)
    assert (parts[..., 3] >= 0.999e-9).all()
    sign = lambda t: np.sign(np.linalg.det(np.stack([t[:, 0] / t[:, 3], t[:, 1] / t[:, 3], np.ones(3)], axis=1)))
    assert all(sign(t) == sign(parts[0]) for t in parts)


def test_mesh_surface_area_known_answers():
    tri = ml.TriangleMesh(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0.0]]), None, np.zeros((3, 2)), np.array([[0, 1, 2]]))
    assert ml.mesh_surface_area(tri) == 0.5
    v = np.array([[x, y, z] for x in (0, 1) for y in (0, 1) for z in (0, 1)], float)
    f = [(0, 1, 3), (0, 3, 2), (4, 6, 7), (4, 7, 5), (0, 4, 5), (0, 5, 1), (2, 3, 7), (2, 7, 6), (0, 2, 6), (0, 6, 4),
         (1, 5, 7), (1, 7, 3)]
    cube = ml.TriangleMesh(v, None, np.zeros((8, 2)), np.array(f))
    assert abs(ml.mesh_surface_area(cube) - 6.0) < 1e-12
    rng = np.random.default_rng(1)
    P = rng.normal(size=(150, 3))
    m = ml.TriangleMesh(P, None, np.zeros((150, 2)), np.arange(150).reshape(50, 3))
    a, b, c = (np.linalg.norm(P[1::3] - P[0::3], axis=1), np.linalg.norm(P[2::3] - P[1::3], axis=1),
               np.linalg.norm(P[0::3] - P[2::3], axis=1))
    s = (a + b + c) / 2
    heron = np.sqrt(s * (s - a) * (s - b) * (s - c)).sum()
    assert abs(ml.mesh_surface_area(m) - heron) <= 1e-9 * heron


def test_synthetic_meshes_have_the_configured_sizes():
    assert synth.icosphere_mesh(5).num_triangles == 20480                        # C1
    m = synth.heightfield_mesh(20)
    assert m.num_triangles == 800 and m.uvs.min() >= 0 and m.uvs.max() <= 1
    assert 2 * 707 * 707 == 999698                                               # C2 triangle count
    assert synth.circle_shape(10).shape == (20, 20) and synth.circle_shape(10).sum() > 300


# ------------------------------------------------------------------ row sharding arithmetic

@pytest.mark.parametrize("height,ws", [(16, 1), (17, 2), (1024, 8), (5, 8), (32768, 8)])
def test_shard_rows_tiles_the_atlas(height, ws):
    slabs = sharding.all_slabs(height, ws)
    assert slabs[0][0] == 0 and sum(r for _, r in slabs) == height
    for (a0, ar), (b0, _) in zip(slabs, slabs[1:]):
        assert a0 + ar == b0
    assert max(r for _, r in slabs) - min(r for _, r in slabs) <= 1
    assert sharding.halo_bounds(0, 4, 16, 2) == (0, 6) and sharding.halo_bounds(12, 4, 16, 2) == (10, 6)
