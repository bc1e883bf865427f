"""mesh_core -- meshes, cameras and the three rasterisation-backed operations of SPEC.md:23-99
(``render_depth`` SPEC:54, ``uv_coverage`` SPEC:63, ``mesh_surface_area`` SPEC:72), plus the
north-star extension ``build_surface_map``.

Host code prepares the small per-triangle arrays (numpy, float64); every per-texel / per-pixel
loop runs in ``libmeshlayers_b200.so`` through ``_native``.  OBJ/PLY loading is out of scope
(configs are synthetic meshes).
"""
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import DegenerateCamera, EmptyMesh, MissingUVs, UVRangeError


@dataclass
class TriangleMesh:
    """SPEC.md:28-34.  Indexed triangles with per-vertex position, normal, uv in [0,1]^2."""
    vertices: np.ndarray          # (V,3) float64
    normals: np.ndarray           # (V,3) float64
    uvs: np.ndarray               # (V,2) float64
    triangles: np.ndarray         # (T,3) int64

    def __post_init__(self):
        self.vertices = np.ascontiguousarray(self.vertices, dtype=np.float64)
        self.triangles = np.ascontiguousarray(self.triangles, dtype=np.int64)
        if self.uvs is None:
            raise MissingUVs("mesh has no texture coordinates")
        self.uvs = np.ascontiguousarray(self.uvs, dtype=np.float64)
        if self.triangles.size and (self.triangles.min() < 0 or self.triangles.max() >= len(self.vertices)):
            raise EmptyMesh("triangle index out of range")
        if self.uvs.size and (self.uvs.min() < 0.0 or self.uvs.max() > 1.0):
            raise UVRangeError("uv outside [0,1]")
        if self.normals is None:
            self.normals = compute_normals(self.vertices, self.triangles)
        self.normals = np.ascontiguousarray(self.normals, dtype=np.float64)

    @property
    def num_triangles(self):
        return int(self.triangles.shape[0])

    @property
    def bbox(self):
        return self.vertices.min(axis=0), self.vertices.max(axis=0)

    # per-triangle arrays in the layout the kernels consume
    def tri_pos(self):
        return np.ascontiguousarray(self.vertices[self.triangles])       # (T,3,3)

    def tri_nrm(self):
        return np.ascontiguousarray(self.normals[self.triangles])        # (T,3,3)

    def tri_uv_texels(self, width, height):
        """uv scaled to grid units (kernels take texel units, y-up)."""
        uv = self.uvs[self.triangles]
        return np.ascontiguousarray(uv * np.array([float(width), float(height)]))


def compute_normals(vertices, triangles):
    """Area-weighted average of incident face normals, normalised."""
    p = vertices[triangles]
    fn = np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0])
    n = np.zeros_like(vertices)
    for k in range(3):
        np.add.at(n, triangles[:, k], fn)
    ln = np.linalg.norm(n, axis=1, keepdims=True)
    return n / np.where(ln > 0, ln, 1.0)


@dataclass
class Camera:
    """SPEC.md:35-38."""
    view: np.ndarray
    projection: np.ndarray
    width: int
    height: int
    generation: int = field(default=0)

    _TRACKED = ("view", "projection", "width", "height")

    def __post_init__(self):
        object.__setattr__(self, "view", np.asarray(self.view, dtype=np.float64).reshape(4, 4))
        object.__setattr__(self, "projection", np.asarray(self.projection, dtype=np.float64).reshape(4, 4))
        self._validate()
        object.__setattr__(self, "_ready", True)

    def _validate(self):
        if self.width < 1 or self.height < 1:
            raise DegenerateCamera("viewport must be at least 1x1")
        m = self.projection @ self.view
        if not np.all(np.isfinite(m)) or abs(np.linalg.det(self.projection)) == 0.0 \
                or abs(np.linalg.det(self.view)) == 0.0:
            raise DegenerateCamera("camera transforms must be finite and invertible")

    def __setattr__(self, name, value):
        """Assigning a new view / projection / viewport after construction is a camera change: the
        generation counter is bumped here, so a depth map or stroke context made for the
        old state is detected as stale without relying on the caller to count."""
        if name in self._TRACKED and getattr(self, "_ready", False):
            if name in ("view", "projection"):
                value = np.asarray(value, dtype=np.float64).reshape(4, 4)
            old = getattr(self, name)
            object.__setattr__(self, name, value)
            try:
                self._validate()
            except DegenerateCamera:
                object.__setattr__(self, name, old)
                raise
            object.__setattr__(self, "generation", self.generation + 1)
            return
        object.__setattr__(self, name, value)

    def set_view(self, view):
        self.view = view
        return self.generation

    def set_projection(self, projection):
        self.projection = projection
        return self.generation

    def state_key(self):
        """Identity of the camera state a depth map / stroke context was derived from: generation,
        viewport and the bytes of MVP (the last catches in-place edits of the matrices)."""
        return (self.generation, int(self.width), int(self.height), self.mvp.tobytes())

    @property
    def mvp(self):
        return self.projection @ self.view

    def clip_coords(self, vertices):
        """(V,4) homogeneous clip coordinates MVP * [x y z 1]."""
        v4 = np.concatenate([vertices, np.ones((vertices.shape[0], 1))], axis=1)
        return v4 @ self.mvp.T


def mesh_surface_area(mesh):
    """sum of cross-product triangle areas (host float64; O(T), not a texel loop)."""
    p = mesh.tri_pos()
    cr = np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0])
    return float(np.sqrt((cr * cr).sum(axis=1)).sum() * 0.5)


def _clip_eye_plane(clip, eps_w):
    """Triangles (T,3,4) in clip space with vertices on both sides of the plane w = eps_w, clipped to
    w >= eps_w (Sutherland-Hodgman against one plane): one triangle when one vertex is inside, two when two
    are.  Vertex order (winding) is preserved."""
    inside = clip[..., 3] > eps_w                                        # (T,3)
    nin = inside.sum(axis=1)
    out = []
    idx = np.arange(3)

    def cut(p_in, p_out):                                               # intersection of edge in -> out with the plane
        t = (p_in[:, 3] - eps_w) / (p_in[:, 3] - p_out[:, 3])
        return p_in + t[:, None] * (p_out - p_in)

    one = np.flatnonzero(nin == 1)
    if one.size:
        k = inside[one].argmax(axis=1)                                  # the inside vertex, rotated to the front
        a = clip[one, k]
        b = clip[one, (k + 1) % 3]
        c = clip[one, (k + 2) % 3]
        out.append(np.stack([a, cut(a, b), cut(a, c)], axis=1))
    two = np.flatnonzero(nin == 2)
    if two.size:
        k = (~inside[two]).argmax(axis=1)                               # the outside vertex c; a, b follow it cyclically
        c = clip[two, k]
        a = clip[two, (k + 1) % 3]
        b = clip[two, (k + 2) % 3]
        bc, ca = cut(b, c), cut(a, c)
        out.append(np.stack([a, b, bc], axis=1))
        out.append(np.stack([a, bc, ca], axis=1))
    del idx
    return np.concatenate(out, axis=0) if out else np.zeros((0, 3, 4))


def window_triangles(mesh, camera):
    """Per-triangle window-space xy (T',3,2) and NDC z (T',3) for the depth pass (KN:106 expects input with
    w > 0).  Triangles entirely behind the eye plane are dropped; triangles CROSSING it are clipped to
    w >= eps_w (1 or 2 triangles, appended after the untouched ones), so geometry that straddles the camera
    still occludes what lies behind its visible part (SPEC 'occlusion safety'; round-1 dropped such triangles
    whole).  Triangles with all three w > 0 pass through unchanged, in order."""
    clip = camera.clip_coords(mesh.vertices)[mesh.triangles]            # (T,3,4)
    w = clip[..., 3]
    keep = (w > 0.0).all(axis=1)
    crossing = (~keep) & (w > 0.0).any(axis=1)
    parts = [clip[keep]]
    if crossing.any():
        eps_w = 1e-9 * float(np.abs(w).max())
        parts.append(_clip_eye_plane(clip[crossing], eps_w))
    clip = np.concatenate(parts, axis=0) if len(parts) > 1 else parts[0]
    ndc = clip[..., :3] / clip[..., 3:4]
    xy = np.empty(clip.shape[:2] + (2,), dtype=np.float64)
    xy[..., 0] = (ndc[..., 0] + 1.0) * 0.5 * camera.width
    xy[..., 1] = (ndc[..., 1] + 1.0) * 0.5 * camera.height
    return np.ascontiguousarray(xy), np.ascontiguousarray(ndc[..., 2])


class DepthMap:
    """float32 plane on the device, 1.0 = background, tagged with the camera
    generation it was rendered for (StaleDepth detection)."""

    def __init__(self, plane, generation, camera_key=None):
        self.plane = plane
        self.generation = generation
        self.camera_key = camera_key          # Camera.state_key() at render time (None: caller-made plane)

    @property
    def shape(self):
        return tuple(self.plane.shape)


def render_depth(mesh, camera, device="cuda"):
    """nearest depth per pixel under the deterministic raster rules."""
    torch = _native.require_cuda()
    depth = torch.ones((camera.height, camera.width), dtype=torch.float32, device=device)
    xy, zn = window_triangles(mesh, camera)
    if xy.shape[0]:
        _native.raster_depth(torch.from_numpy(xy).to(device), torch.from_numpy(zn).to(device), depth, count=False)
    return DepthMap(depth, camera.generation, camera.state_key())


def uv_coverage(mesh, resolution, device="cuda"):
    """bool grid, true iff the texel centre is covered by a uv triangle."""
    torch = _native.require_cuda()
    w, h = (resolution, resolution) if np.isscalar(resolution) else resolution
    out = torch.zeros((h, w), dtype=torch.uint8, device=device)
    if mesh.num_triangles:
        _native.coverage_fill(torch.from_numpy(mesh.tri_uv_texels(w, h)).to(device), w, h, out)
    return out.view(torch.bool)


class SurfaceMap:
    """Per-texel 3D position / normal / area / owner-triangle map of one atlas row slab
    (north star (1)).  ``overlap`` > 0 flags overlapping uv islands (SPEC.md:99 diagnostic)."""

    def __init__(self, fields, width, height, row0, tri_xy):
        self.tri_id, self.pos, self.nrm, self.area = (fields[k] for k in ("tri_id", "pos", "nrm", "area"))
        self.covered, self.fragments, self.overlap = fields["covered"], fields["fragments"], fields["overlap"]
        self.width, self.height, self.row0 = width, height, row0
        self.rows = int(self.tri_id.shape[0])
        self.tri_xy = tri_xy                                    # device (T,3,2), reused by TEA
        # per-tile position boxes for the footprint-culled sphere brushes (None: width % 128 != 0)
        self.tiles = _native.tile_boxes(self.pos)

    @property
    def coverage(self):
        return self.tri_id >= 0


def build_surface_map(mesh, width, height, *, row0=0, rows=None, device="cuda"):
    """Rasterise every triangle into the atlas (uv as position) and interpolate position,
    normal and per-texel area for the owner triangle (definition: oracle ext_surface_map)."""
    torch = _native.require_cuda()
    if mesh.num_triangles == 0:
        raise EmptyMesh("mesh has no triangles")
    tri_xy = torch.from_numpy(mesh.tri_uv_texels(width, height)).to(device)
    fields = _native.surface_map(tri_xy, mesh.tri_pos(), mesh.tri_nrm(), width, height,
                                 row0=row0, rows=rows, device=device)
    return SurfaceMap(fields, width, height, row0, tri_xy)
