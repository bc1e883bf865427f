"""raster_device -- pooled texture planes in HBM (thin slice).

``TexturePool`` is the reference's pool keyed by (width, height, kind): planes
are zero-initialised torch CUDA tensors, freed slots are reused under the same key, allocation is
deferred until the first acquire of a key, and a global texel budget (default 512 Mtexels,
SPEC.md:147) raises ``CapacityExceeded``.  On a 180 GB B200 the budget is the only limit that
matters; raise it explicitly for 16k^2 x 64-layer workloads.
"""
import os

from . import _native
from .errors import CapacityExceeded, TargetMismatch

#: SPEC.md:107 element kinds -> torch dtype names.  ``rgba8`` planes are uint8 with a trailing 4.
KINDS = ("int8", "int16", "int32", "uint8", "uint32", "float16", "float32", "bool", "rgba8")

DEFAULT_BUDGET_TEXELS = 512 * 1024 * 1024


def _torch_dtype(kind):
    torch = _native._torch()
    table = {"int8": torch.int8, "int16": torch.int16, "int32": torch.int32, "uint8": torch.uint8,
             "uint32": torch.uint32, "float16": torch.float16, "float32": torch.float32,
             "bool": torch.bool, "rgba8": torch.uint8}
    if kind not in table:
        raise TargetMismatch("unknown plane kind %r" % (kind,))
    return table[kind]


class PlaneHandle:
    """A pooled plane: ``tensor`` is the device storage, valid until released."""

    __slots__ = ("pool", "key", "slot", "tensor")

    def __init__(self, pool, key, slot, tensor):
        self.pool, self.key, self.slot, self.tensor = pool, key, slot, tensor

    @property
    def kind(self):
        return self.key[2]

    def release(self):
        self.pool.release(self)


class TexturePool:
    def __init__(self, budget_texels=None, device="cuda"):
        env = os.environ.get("MESHLAYERS_TEXEL_BUDGET")             # SPEC.md:493 env variable
        self.budget = int(budget_texels if budget_texels is not None else (env or DEFAULT_BUDGET_TEXELS))
        self.device = device
        self._planes = {}        # key -> list of tensors (None = never used)
        self._free = {}          # key -> list of free slot indices
        self.texels_in_use = 0

    @property
    def keys(self):
        return list(self._planes)

    def plane_count(self, key):
        return len(self._planes.get(key, ()))

    def acquire(self, width, height, kind):
        """SPEC.md:120-128 ``pool_acquire``."""
        torch = _native.require_cuda()
        if width < 1 or height < 1:
            raise TargetMismatch("plane dimensions must be >= 1")
        key = (int(width), int(height), kind)
        dtype = _torch_dtype(kind)
        free = self._free.setdefault(key, [])
        planes = self._planes.setdefault(key, [])
        if free:
            slot = free.pop()
            t = planes[slot]
            t.zero_()                                                # SPEC.md:128 contents zeroed
        else:
            if self.texels_in_use + width * height > self.budget:
                if not planes:
                    del self._planes[key]
                    del self._free[key]
                raise CapacityExceeded("texel budget of %d exceeded" % self.budget)
            shape = (height, width, 4) if kind == "rgba8" else (height, width)
            t = torch.zeros(shape, dtype=dtype, device=self.device)
            planes.append(t)
            slot = len(planes) - 1
            self.texels_in_use += width * height
        return PlaneHandle(self, key, slot, t)

    def release(self, handle):
        self._free[handle.key].append(handle.slot)


_default_pool = None


def default_pool():
    global _default_pool
    if _default_pool is None:
        _default_pool = TexturePool()
    return _default_pool


def pool_acquire(width, height, kind, pool=None):
    """Module-level spelling of SPEC.md:120."""
    return (pool or default_pool()).acquire(width, height, kind)


def rasterize(tri_xy, targets, values, keep=None):
    """SPEC.md:129-137 ``rasterize`` for the fragment rules a device backend can take without a
    host callback: every texel whose centre lies inside a triangle (top-left rule, RasterRules) is
    offered to the rule "triangle t keeps its fragments iff keep[t], and writes values[k][t] into
    target k"; writes are atomic per texel and the last triangle in submission order wins on overlap
    (SPEC.md:132).  ``tri_xy`` (T,3,2) in texel units; ``targets`` a list of plane handles / CUDA
    tensors sharing dimensions; ``values`` one scalar or (T,) array per target; ``keep`` an optional
    (T,) bool array ("always discard" = all False).  Returns the count of written texels."""
    torch = _native.require_cuda()
    planes = [t.tensor if isinstance(t, PlaneHandle) else t for t in targets]
    if not planes:
        return 0
    shape = tuple(planes[0].shape[:2])
    if any(tuple(p.shape[:2]) != shape for p in planes):
        raise TargetMismatch("targets disagree in dimensions")
    import numpy as np
    T = int(tri_xy.shape[0])
    if T == 0:
        return 0
    dev = planes[0].device
    # Fragments are offered to the rule triangle by triangle and the LAST KEPT write wins: a texel
    # covered by a kept triangle and by a later discarded one holds the kept triangle's value.  So the discarded
    # triangles are dropped BEFORE the owner pass (an owner map over all triangles followed by a keep test would
    # leave such texels unwritten); values are gathered with the same selection, which keeps submission order.
    sel = None
    if keep is not None:
        sel = np.flatnonzero(np.asarray(keep).astype(bool).reshape(T))
        if sel.size == 0:
            return 0
        if torch.is_tensor(tri_xy):
            tri_xy = tri_xy[torch.from_numpy(sel).to(tri_xy.device)]
        else:
            tri_xy = np.ascontiguousarray(np.asarray(tri_xy)[sel])
    tri_id, _, _ = _native.raster_tri_id(tri_xy, shape[1], shape[0], device=dev)
    written = 0
    for plane, vals in zip(planes, values):
        dt = _native._np_dtype_of(plane)
        v = np.broadcast_to(np.asarray(vals).astype(dt), (T,))
        v = np.ascontiguousarray(v if sel is None else v[sel])
        vt = torch.from_numpy(v.view({1: np.uint8, 2: np.int16, 4: np.int32}[dt.itemsize])).to(dev)
        written = _native.owner_values(tri_id, vt, plane, None)
    return written
