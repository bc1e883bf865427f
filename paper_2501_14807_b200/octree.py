"""octree_baseline -- the OCT-TR layer scheme the paper benchmarks against, on the
B200 kernels of ``csrc/octree.cu``: a surface-crossing octree built level by level with
``expand_pairs_ordered`` (KN:303), per-leaf layer values, editing by per-pixel ray casting with
``raycast`` (KN:361), and the simulated colour re-upload accounting (4 bytes per crossed leaf).

The reference ships the two kernels but not this caller; the operations follow SPEC.md
and keep its names: ``build_octree``, ``octree_edit``, ``octree_upload_size``, ``octree_precision``.
Everything stays on the device; there is no CPU fallback.
"""
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import MemoryBudgetExceeded, TargetMismatch

#: bytes per (leaf, triangle) row while a level is being built: the emitted cell (12) + triangle (4),
#: its Morton key (8), the sort permutation (8) and the next level's parent index (4)
ROW_BYTES = 36
MAX_DEPTH = 16


@dataclass
class SurfaceOctree:
    """SPEC.md:332-335.  Leaves at depth ``depth`` crossed by the surface, as the arrays ``raycast``
    consumes: sorted Morton ``keys`` (canonical depth-first octant order), CSR
    ``offsets`` into ``tri_idx`` (triangle indices ascending inside a leaf)."""
    depth: int
    cube_min: np.ndarray            # (3,) float64
    side: float
    keys: object                    # (L,) int64 CUDA, sorted
    offsets: object                 # (L+1,) int64 CUDA
    tri_idx: object                 # (P,) int32 CUDA
    coarse: object                  # (2^cb,)*3 uint8 CUDA occupancy of the cells >> coarse_shift
    coarse_shift: int
    verts: object                   # (V,3) float64 CUDA
    tris: object                    # (T,3) int32 CUDA
    node_count: int = 0
    level_cells: tuple = ()
    build_ms: float = 0.0
    peak_bytes: int = 0

    @property
    def n_cells(self):
        return 1 << self.depth

    @property
    def h(self):
        return self.side / float(self.n_cells)

    @property
    def leaf_count(self):
        return int(self.keys.shape[0])

    def leaf_cells(self):
        """(L,3) integer coordinates of the leaves (Morton decode), CUDA int64."""
        torch = _native._torch()

        def compact(v):
            v = v & 0x1249249249249249
            for sh, m in ((2, 0x10c30c30c30c30c3), (4, 0x100f00f00f00f00f), (8, 0x1f0000ff0000ff),
                          (16, 0x1f00000000ffff), (32, 0x1fffff)):
                v = (v | (v >> sh)) & m
            return v
        k = self.keys
        return torch.stack([compact(k), compact(k >> 1), compact(k >> 2)], 1)


@dataclass
class OctreeLayer:
    """one value + validity flag per crossed leaf, in the octree's key order."""
    values: object
    valid: object
    kind: str = "uint8"

    @property
    def leaf_count(self):
        return int(self.values.shape[0])


@dataclass
class OctreeEditResult:
    """edited leaf set (indices into the octree's key order), rays cast, transfer bytes."""
    edited_leaves: object
    _rays: object
    _hits: object
    transfer_bytes: int
    duration_ms: float = 0.0
    _cache: dict = field(default_factory=dict)

    @property
    def edited_count(self):
        return int(self.edited_leaves.shape[0])

    @property
    def rays(self):
        """Rays cast = window pixels inside the tool shape (read from the device on demand)."""
        return int(self._rays)

    @property
    def hits(self):
        """Rays whose nearest hit lies in a leaf of the octree (read from the device on demand)."""
        return int(self._hits)


def bounding_cube(vertices, pad=1e-3):
    """Root cube: the mesh bounding box cubified to its largest extent, padded by
    ``pad`` so that no vertex lies on the outer faces."""
    lo, hi = vertices.min(0), vertices.max(0)
    side = float((hi - lo).max()) * (1.0 + pad)
    if not side > 0.0:
        side = 1.0
    centre = 0.5 * (lo + hi)
    return np.ascontiguousarray(centre - 0.5 * side, dtype=np.float64), side


def build_octree(mesh, depth, *, budget_bytes=0, coarse_bits=8, cube=None, device="cuda"):
    """SPEC.md:342-349.  Level-by-level refinement: every (cell, triangle) pair of level k-1 is tested
    against the 8 child cubes (closed-box SAT, touching counts); children crossed by no
    triangle never exist.  ``budget_bytes`` > 0 raises ``MemoryBudgetExceeded`` as soon as a level's
    working set would exceed it (acceptance #11) -- before the level is materialised."""
    torch = _native.require_cuda()
    depth = int(depth)
    if not 0 <= depth <= MAX_DEPTH:
        raise TargetMismatch("octree depth must be in [0, %d]" % MAX_DEPTH)
    T = mesh.num_triangles
    if T < 1:
        raise TargetMismatch("build_octree needs a non-empty mesh")
    cube_min, side = cube if cube is not None else bounding_cube(mesh.vertices)
    cube_min = np.ascontiguousarray(cube_min, dtype=np.float64)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    verts = torch.from_numpy(mesh.vertices).to(device)
    tris = torch.from_numpy(mesh.triangles.astype(np.int32)).to(device)
    base_bytes = verts.numel() * 8 + tris.numel() * 4
    max_rows = None
    if budget_bytes:
        max_rows = max(0, (int(budget_bytes) - base_bytes)) // ROW_BYTES
        if T > max_rows:
            raise MemoryBudgetExceeded("octree root needs %d rows, the budget allows %d" % (T, max_rows))
    cells = torch.zeros((T, 3), dtype=torch.int32, device=device)
    pair_tri = torch.arange(T, dtype=torch.int32, device=device)
    parent_cells = torch.zeros((1, 3), dtype=torch.int32, device=device)
    pair_parent = torch.zeros(T, dtype=torch.int32, device=device)
    key = torch.zeros(T, dtype=torch.int64, device=device)
    nodes, level_cells, peak_rows = 1, [1], T
    for lvl in range(1, depth + 1):
        child_h = side / float(1 << lvl)
        cells, pair_tri = _native.expand_pairs_ordered(verts, tris, parent_cells, pair_parent, pair_tri,
                                                       cube_min, child_h, max_rows=max_rows)
        key = _native.morton_encode(cells[:, 0], cells[:, 1], cells[:, 2])
        ukeys, inverse = torch.unique(key, return_inverse=True)
        first = torch.full((ukeys.shape[0],), key.shape[0], dtype=torch.int64, device=device)
        first.scatter_reduce_(0, inverse, torch.arange(key.shape[0], device=device), "amin")
        parent_cells = cells[first].contiguous()
        pair_parent = inverse.to(torch.int32)
        nodes += int(ukeys.shape[0])
        level_cells.append(int(ukeys.shape[0]))
        peak_rows = max(peak_rows, int(key.shape[0]))
    # leaves: rows sorted by (key, triangle index)
    order = torch.argsort(pair_tri, stable=True)
    order = order[torch.argsort(key[order], stable=True)]
    keys, counts = torch.unique_consecutive(key[order], return_counts=True)
    offsets = torch.zeros(keys.shape[0] + 1, dtype=torch.int64, device=device)
    offsets[1:] = torch.cumsum(counts, 0)
    tri_idx = pair_tri[order].contiguous()
    cb = min(int(coarse_bits), depth)
    shift = depth - cb
    coarse = torch.zeros((1 << cb,) * 3, dtype=torch.uint8, device=device)
    lc = cells.to(torch.int64) >> shift
    coarse[lc[:, 0], lc[:, 1], lc[:, 2]] = 1
    b.record()
    torch.cuda.synchronize()
    return SurfaceOctree(depth=depth, cube_min=cube_min, side=side, keys=keys.contiguous(), offsets=offsets,
                         tri_idx=tri_idx, coarse=coarse, coarse_shift=shift, verts=verts, tris=tris,
                         node_count=nodes, level_cells=tuple(level_cells), build_ms=a.elapsed_time(b),
                         peak_bytes=base_bytes + peak_rows * ROW_BYTES)


def create_octree_layer(octree, kind="uint8", device="cuda"):
    """An empty OctreeLayer over the octree's crossed leaves."""
    torch = _native.require_cuda()
    dt = getattr(torch, kind)
    n = octree.leaf_count
    return OctreeLayer(values=torch.zeros(n, dtype=dt, device=device),
                       valid=torch.zeros(n, dtype=torch.bool, device=device), kind=kind)


def tool_rays(camera, tool, device=None):
    """One ray per window pixel inside the tool shape: pixel centres through the inverse
    view-projection, origin on the near plane, unit direction; float64 (N,3).  A pixel is inside the
    tool when its centre maps into the tool bitmap through the texture engine's own tool map
    (KN:187-193 with the factors of ``compute_tool_projection``; half-open at the far edges so that a
    (2r+1)-pixel square covers (2r+1)^2 pixels): both engines edit under one footprint.
    ``device=None`` returns numpy arrays, otherwise the rays are generated on that device (torch)."""
    torch = _native._torch()
    if device is not None and torch.device(device).type == "cuda":
        o, d, _ = _tool_rays_padded(camera, tool, device)          # the rays octree_edit casts, compacted
        keep = ~torch.isnan(d[:, 0])
        return o[keep].contiguous(), d[keep].contiguous()
    dev = device if device is not None else "cpu"
    shape = tool.shape if type(tool.shape).__module__.startswith("torch") else torch.from_numpy(
        np.ascontiguousarray(tool.shape))
    shape = shape.to(dev)
    th, tw = int(shape.shape[0]), int(shape.shape[1])
    left, bottom = tool.px - 0.5 * tw, tool.py - 0.5 * th
    x0, x1 = max(0, int(np.floor(left))), min(camera.width, int(np.ceil(left + tw)) + 1)
    y0, y1 = max(0, int(np.floor(bottom))), min(camera.height, int(np.ceil(bottom + th)) + 1)
    if x1 <= x0 or y1 <= y0:
        z = torch.zeros((0, 3), dtype=torch.float64, device=dev)
        return (z, z.clone()) if device is not None else (z.numpy(), z.clone().numpy())
    xs = torch.arange(x0, x1, dtype=torch.float64, device=dev) + 0.5
    ys = torch.arange(y0, y1, dtype=torch.float64, device=dev) + 0.5
    gy, gx = torch.meshgrid(ys, xs, indexing="ij")
    s, t = (gx - left) / tw, (gy - bottom) / th                     # the tool map of KN:187-192 per pixel
    inside = (s >= 0.0) & (s < 1.0) & (t >= 0.0) & (t < 1.0)        # half open: (2r+1)^2 pixels
    si = (s * tw).to(torch.int64).clamp_(0, tw - 1)
    ti = (t * th).to(torch.int64).clamp_(0, th - 1)
    keep = inside & (shape[ti, si] != 0)
    x, y = gx[keep], gy[keep]
    inv = torch.from_numpy(np.linalg.inv(np.asarray(camera.mvp, dtype=np.float64))).to(dev)
    one = torch.ones_like(x)
    nx, ny = x / camera.width * 2.0 - 1.0, y / camera.height * 2.0 - 1.0
    near = torch.stack([nx, ny, -one, one], 1) @ inv.T
    far = torch.stack([nx, ny, one, one], 1) @ inv.T
    near, far = near[:, :3] / near[:, 3:], far[:, :3] / far[:, 3:]
    d = far - near
    d = d / torch.linalg.norm(d, dim=1, keepdim=True)
    near, d = near.contiguous(), d.contiguous()
    return (near, d) if device is not None else (near.numpy(), d.numpy())


def _tool_rays_padded(camera, tool, device):
    """Device-side ray set-up (``ml_tool_rays``): rays for EVERY pixel of the tool's window box, pixels outside
    the tool shape carrying a NaN direction (a miss for ``raycast``); returns (origins, dirs, count tensor)."""
    import ctypes as C
    torch = _native.require_cuda()
    shape = _native._as_dev_bytes(tool.shape, device)
    th, tw = int(shape.shape[0]), int(shape.shape[1])
    left, bottom = tool.px - 0.5 * tw, tool.py - 0.5 * th
    x0, x1 = max(0, int(np.floor(left))), min(camera.width, int(np.ceil(left + tw)) + 1)
    y0, y1 = max(0, int(np.floor(bottom))), min(camera.height, int(np.ceil(bottom + th)) + 1)
    nx, ny = max(0, x1 - x0), max(0, y1 - y0)
    origins = torch.empty((nx * ny, 3), dtype=torch.float64, device=device)
    dirs = torch.empty((nx * ny, 3), dtype=torch.float64, device=device)
    count = torch.zeros(1, dtype=torch.int64, device=device)
    inv = np.ascontiguousarray(np.linalg.inv(np.asarray(camera.mvp, dtype=np.float64)))
    _native._check(_native.lib().ml_tool_rays(inv.ctypes.data, camera.width, camera.height, float(tool.px),
                                              float(tool.py), _native._ptr(shape), tw, th, x0, y0, nx, ny,
                                              _native._ptr(origins), _native._ptr(dirs), _native._ptr(count),
                                              _native._stream()))
    return origins, dirs, count


def octree_edit(octree, layer, mesh, camera, tool, value=None):
    """cast the camera ray of every window pixel inside the tool shape, take the
    nearest ray-triangle hit (front-to-back DDA, KN:361) and set the value and validity of the leaf
    that contains the hit point.  ``mesh`` is the mesh the octree was built over (its arrays already
    live in ``octree``)."""
    torch = _native.require_cuda()
    if layer.leaf_count != octree.leaf_count:
        raise TargetMismatch("layer has %d leaves, the octree %d" % (layer.leaf_count, octree.leaf_count))
    dev = octree.keys.device
    origins, dirs, n = _tool_rays_padded(camera, tool, dev)
    if origins.shape[0] == 0:
        empty = torch.zeros(0, dtype=torch.int64, device=dev)
        return OctreeEditResult(empty, 0, 0, octree_upload_size(layer))
    best_t, best_tri, leaf = _native.raycast(origins, dirs, octree.keys, octree.offsets, octree.tri_idx, octree.verts,
                                             octree.tris, octree.cube_min, octree.h, octree.n_cells,
                                             octree.coarse, octree.coarse_shift, None)
    hit = leaf >= 0
    leaves = torch.unique(leaf[hit])
    v = tool.value if value is None else value
    layer.values[leaves] = torch.as_tensor(v).to(layer.values.dtype).to(dev)
    layer.valid[leaves] = True
    return OctreeEditResult(leaves, n, hit.sum(), octree_upload_size(layer))


def octree_upload_size(layer):
    """crossed-leaf count x 4 bytes (RGBA8 per leaf), the simulated full-layer colour
    re-upload per edit.  Accepts an OctreeLayer, a SurfaceOctree or a leaf count."""
    n = layer if isinstance(layer, int) else layer.leaf_count
    return 4 * int(n)


def octree_precision(octree, mesh, units_to_cm=100.0):
    """mesh surface area / crossed-leaf count, in cm^2."""
    from .mesh_core import mesh_surface_area
    if octree.leaf_count == 0:
        return None
    return mesh_surface_area(mesh) * units_to_cm ** 2 / octree.leaf_count
