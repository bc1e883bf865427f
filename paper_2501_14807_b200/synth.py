"""Deterministic synthetic meshes, atlases, cameras and strokes (SURVEY.md 8(d) inputs).

Host-side numpy only: these build the *inputs* of the hot path (there is no network for real
datasets).  Used by tests, ``bench.py`` and ``__graft_entry__.smoke()``.
"""
import math

import numpy as np

from .mesh_core import Camera, TriangleMesh

SEED = 2501_14807


# --------------------------------------------------------------------------------------------
# meshes

def icosphere(level):
    """Unit icosphere, `level` subdivisions: 20*4^level triangles (level 5 -> 20,480)."""
    t = (1.0 + math.sqrt(5.0)) / 2.0
    v = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t),
         (0, -1, -t), (0, 1, -t), (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    f = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
         (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8),
         (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    verts = [np.array(p, dtype=np.float64) / math.sqrt(1 + t * t) for p in v]
    faces = list(f)
    for _ in range(level):
        cache = {}
        new_faces = []

        def mid(a, b):
            key = (a, b) if a < b else (b, a)
            if key not in cache:
                m = verts[a] + verts[b]
                verts.append(m / np.linalg.norm(m))
                cache[key] = len(verts) - 1
            return cache[key]

        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            new_faces += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = new_faces
    return np.array(verts, dtype=np.float64), np.array(faces, dtype=np.int64)


def chart_grid_mesh(verts, faces, normals=None, gutter_frac=0.1):
    """Unweld the mesh and give every triangle its own island: "two triangles per square cell"
    chart grid with a gutter, no overlaps (SURVEY.md 8(d) C1 atlas)."""
    T = faces.shape[0]
    cells = (T + 1) // 2
    side = int(math.ceil(math.sqrt(cells)))
    cell = 1.0 / side
    g = gutter_frac * cell
    k = np.arange(T)
    ci = k // 2
    cx = (ci % side).astype(np.float64) * cell
    cy = (ci // side).astype(np.float64) * cell
    lower = (k % 2) == 0
    lo, hi = g, cell - g
    # lower-left and upper-right triangles of the cell, separated by a diagonal gutter
    uv = np.empty((T, 3, 2), dtype=np.float64)
    d = 0.5 * g
    uv[:, 0, 0] = np.where(lower, cx + lo, cx + hi)
    uv[:, 0, 1] = np.where(lower, cy + lo, cy + hi)
    uv[:, 1, 0] = np.where(lower, cx + hi - d - g, cx + lo + d + g)
    uv[:, 1, 1] = np.where(lower, cy + lo, cy + hi)
    uv[:, 2, 0] = np.where(lower, cx + lo, cx + hi)
    uv[:, 2, 1] = np.where(lower, cy + hi - d - g, cy + lo + d + g)
    P = verts[faces]                                        # (T,3,3)
    N = (verts if normals is None else normals)[faces]
    return TriangleMesh(vertices=P.reshape(-1, 3).copy(), normals=N.reshape(-1, 3).copy(),
                        uvs=uv.reshape(-1, 2).copy(),
                        triangles=np.arange(3 * T, dtype=np.int64).reshape(T, 3))


def icosphere_mesh(level=5):
    """C1 mesh: icosphere level 5 -> 20,480 triangles, one uv island per triangle."""
    v, f = icosphere(level)
    return chart_grid_mesh(v, f, normals=v)


def heightfield_mesh(nq, seed=SEED, margin=0.0):
    """C2/C5 mesh: nq x nq quads over [0,1]^2 -> 2*nq^2 triangles, z = 0.1 sin(7x) cos(5y) + noise,
    uv = grid parametrisation (single island, no overlap).  nq=707 -> 999,698 triangles."""
    n = nq + 1
    rng = np.random.default_rng(seed)
    u = np.linspace(0.0, 1.0, n)
    X, Y = np.meshgrid(u, u, indexing="xy")
    Z = 0.1 * np.sin(7.0 * X) * np.cos(5.0 * Y) + 0.002 * rng.standard_normal((n, n))
    verts = np.stack([X, Y, Z], axis=-1).reshape(-1, 3)
    # analytic-ish normals from central differences
    dzdx = np.gradient(Z, u, axis=1)
    dzdy = np.gradient(Z, u, axis=0)
    nr = np.stack([-dzdx, -dzdy, np.ones_like(Z)], axis=-1)
    nr /= np.linalg.norm(nr, axis=-1, keepdims=True)
    uv = np.stack([margin + (1 - 2 * margin) * X, margin + (1 - 2 * margin) * Y], axis=-1).reshape(-1, 2)
    i, j = np.meshgrid(np.arange(nq), np.arange(nq), indexing="xy")
    v00 = (j * n + i).ravel()
    v10, v01, v11 = v00 + 1, v00 + n, v00 + n + 1
    tris = np.concatenate([np.stack([v00, v10, v11], 1), np.stack([v00, v11, v01], 1)], axis=1).reshape(-1, 3)
    return TriangleMesh(vertices=verts, normals=nr.reshape(-1, 3), uvs=uv, triangles=tris.astype(np.int64))


def coaxial_quads_mesh():
    """SPEC.md:285 / 606 occlusion scene: two coaxial quads facing +z, front at z=0.5 (uv left
    half) and back at z=-0.5 (uv right half)."""
    P, uv = [], []
    for z, u0 in ((0.5, 0.02), (-0.5, 0.52)):
        P += [(-1, -1, z), (1, -1, z), (1, 1, z), (-1, 1, z)]
        uv += [(u0, 0.02), (u0 + 0.46, 0.02), (u0 + 0.46, 0.98), (u0, 0.98)]
    tris = [(0, 1, 2), (0, 2, 3), (4, 5, 6), (4, 6, 7)]
    N = [(0, 0, 1)] * 8
    return TriangleMesh(vertices=np.array(P, np.float64), normals=np.array(N, np.float64),
                        uvs=np.array(uv, np.float64), triangles=np.array(tris, np.int64))


def flat_square_mesh(side=1.0):
    """SPEC.md:539 / acceptance #8: flat square of ``side`` units in the z=0 plane whose uv chart fills
    the whole atlas, so every texel is covered and precision = side^2 / resolution^2."""
    P = [(0.0, 0.0, 0.0), (side, 0.0, 0.0), (side, side, 0.0), (0.0, side, 0.0)]
    uv = [(0.0, 0.0), (1.0, 0.0), (1.0, 1.0), (0.0, 1.0)]
    return TriangleMesh(vertices=np.array(P, np.float64), normals=np.array([(0, 0, 1)] * 4, np.float64),
                        uvs=np.array(uv, np.float64), triangles=np.array([(0, 1, 2), (0, 2, 3)], np.int64))


def random_soup(rng, ntri, extent, dtype=np.float64, degenerate_frac=0.05, snap_frac=0.3):
    """Random overlapping triangle soup in grid units for rasteriser parity tests: mixes sizes,
    windings, vertices snapped to texel centres / corners (tie-rule stress) and degenerates."""
    c = rng.uniform(-0.1 * extent, 1.1 * extent, size=(ntri, 1, 2))
    scale = np.exp(rng.uniform(np.log(0.3), np.log(0.35 * extent), size=(ntri, 1, 1)))
    tri = c + rng.normal(size=(ntri, 3, 2)) * scale
    snap = rng.random(ntri) < snap_frac
    tri[snap] = np.round(tri[snap] * 2.0) / 2.0               # half-integers: centres and corners
    deg = rng.random(ntri) < degenerate_frac
    tri[deg, 2] = tri[deg, 1]                                   # zero area
    return tri.astype(dtype)


# --------------------------------------------------------------------------------------------
# cameras / tools

def look_at(eye, target, up=(0.0, 1.0, 0.0)):
    eye, target, up = (np.asarray(a, dtype=np.float64) for a in (eye, target, up))
    f = target - eye
    f /= np.linalg.norm(f)
    s = np.cross(f, up)
    s /= np.linalg.norm(s)
    u = np.cross(s, f)
    m = np.eye(4)
    m[0, :3], m[1, :3], m[2, :3] = s, u, -f
    m[:3, 3] = -m[:3, :3] @ eye
    return m


def perspective(fovy_deg, aspect, near, far):
    f = 1.0 / math.tan(math.radians(fovy_deg) / 2.0)
    m = np.zeros((4, 4))
    m[0, 0], m[1, 1] = f / aspect, f
    m[2, 2], m[2, 3] = (far + near) / (near - far), 2.0 * far * near / (near - far)
    m[3, 2] = -1.0
    return m


def default_camera(width=512, height=512, eye=(0.0, 0.0, 3.0), target=(0.0, 0.0, 0.0), fovy=45.0,
                   near=0.5, far=10.0):
    """C1 camera: at z=+3 looking at the origin, 45 deg fovy, near .5 / far 10, 512^2 window."""
    return Camera(view=look_at(eye, target), projection=perspective(fovy, width / height, near, far),
                  width=width, height=height)


def circle_shape(radius_px):
    """Circular tool shape plane of side 2*radius (SPEC.md:320 built-in generator)."""
    n = max(1, int(2 * radius_px))
    c = (np.arange(n) + 0.5) - n / 2.0
    return ((c[None, :] ** 2 + c[:, None] ** 2) <= float(radius_px) ** 2).astype(np.uint8)


def square_shape(side_px):
    return np.ones((max(1, int(side_px)),) * 2, dtype=np.uint8)


def sphere_strokes(mesh, count, seed=SEED, rmin_frac=0.005, rmax_frac=0.05):
    """C2 strokes: centres at seeded random vertices, radii log-uniform in [0.5%, 5%] of the
    bbox diagonal, labels 1..255 cyclic.  Returns (strokes (K,4) f64, labels (K,) uint8)."""
    rng = np.random.default_rng(seed + 1)
    lo, hi = mesh.vertices.min(0), mesh.vertices.max(0)
    diag = float(np.linalg.norm(hi - lo))
    idx = rng.integers(0, mesh.vertices.shape[0], size=count)
    r = np.exp(rng.uniform(math.log(rmin_frac * diag), math.log(rmax_frac * diag), size=count))
    strokes = np.concatenate([mesh.vertices[idx], r[:, None]], axis=1).astype(np.float64)
    labels = (np.arange(count) % 255 + 1).astype(np.uint8)
    return strokes, labels
