"""layer_core -- information layers on pooled planes (data model only) plus the
north-star extensions the reference leaves out of scope: layer algebra
(``layer_union`` / ``layer_intersection`` / ``layer_difference`` / ``layer_mask`` /
``layer_chain``) and per-layer measurement (``layer_area``, ``layers_area``, ``label_area``,
``layer_stats``).  Palette / display / file format are not part of the hot path.
"""
from . import _native
from .errors import TargetMismatch
from .raster_device import default_pool

NUMERIC_KINDS = ("int8", "int16", "int32", "uint8", "float16", "float32")


class InformationLayer:
    """data plane + bool mask plane (+ display limits).  ``kind`` is one of
    NUMERIC_KINDS or "uint32" for database layers."""

    def __init__(self, name, kind, data_handle, mask_handle, limits=(0.0, 1.0), table=None, palette=None):
        if not limits[0] < limits[1]:
            raise TargetMismatch("layer limits must satisfy lower < upper")
        from .display import Palette
        self.name, self.kind, self.limits, self.table = name, kind, tuple(limits), table
        self.palette = palette if palette is not None else Palette.grayscale()
        self._data_handle, self._mask_handle = data_handle, mask_handle

    @property
    def data(self):
        return self._data_handle.tensor

    @property
    def mask(self):
        return self._mask_handle.tensor

    @property
    def shape(self):
        return tuple(self.mask.shape)

    @property
    def width(self):
        return int(self.mask.shape[1])

    @property
    def height(self):
        return int(self.mask.shape[0])

    def valid_texels(self):
        return int(self.mask.sum().item())

    def release(self):
        self._data_handle.release()
        self._mask_handle.release()


def create_layer(name, kind, width, height, palette=None, limits=(0.0, 1.0), pool=None, table=None):
    """data plane zeroed, mask all-false.  ``height`` may be a row-slab height."""
    if kind not in NUMERIC_KINDS + ("uint32",):
        raise TargetMismatch("unsupported layer kind %r" % (kind,))
    pool = pool or default_pool()
    data = pool.acquire(width, height, kind)
    try:
        mask = pool.acquire(width, height, "bool")
    except Exception:
        data.release()
        raise
    return InformationLayer(name, kind, data, mask, limits=limits, table=table, palette=palette)


def _check_pair(a, b, out):
    if a.shape != b.shape or a.shape != out.shape:
        raise TargetMismatch("layers disagree in dimensions")
    if a.kind != out.kind:
        raise TargetMismatch("output layer kind differs from operand A")


def _binary(op, a, b, out):
    out = a if out is None else out
    _check_pair(a, b, out)
    db = b.data if (b.kind == a.kind) else None
    if op == "union" and db is None:
        raise TargetMismatch("union needs layers of the same kind")
    _native.layer_op(op, a.data, a.mask, db, b.mask, out.data, out.mask)
    return out


def layer_union(a, b, out=None):
    """mask = a|b; data = a where a is valid, else b (A takes precedence)."""
    return _binary("union", a, b, out)


def layer_intersection(a, b, out=None):
    """mask = a&b; data = a there, 0 elsewhere."""
    return _binary("intersection", a, b, out)


def layer_difference(a, b, out=None):
    """mask = a&~b; data = a there, 0 elsewhere."""
    return _binary("difference", a, b, out)


def layer_mask(a, selector, out=None):
    """Masking: keep A where the selector plane (a layer's mask or any byte plane) is non-zero."""
    out = a if out is None else out
    sel = selector.mask if isinstance(selector, InformationLayer) else selector
    if tuple(sel.shape) != a.shape or a.shape != out.shape:
        raise TargetMismatch("layers disagree in dimensions")
    _native.layer_op("masking", a.data, a.mask, None, sel, out.data, out.mask)
    return out


def layer_chain(layers, ops, out, *, lazy=True):
    """((L0 ops[0] L1) ops[1] L2) ... in ONE pass over the atlas (reads N layers, writes 1).
    ``ops`` has len(layers)-1 entries from {"union","intersection","difference","masking"}.
    ``lazy`` (default): data planes of 3..8 one-byte layers are read only where the masks let them
    reach the result; ``lazy=False`` streams every plane (same result)."""
    if len(ops) != len(layers) - 1:
        raise TargetMismatch("need one operator between each pair of layers")
    for l in layers:
        if l.shape != out.shape or l.kind != out.kind:
            raise TargetMismatch("chain layers must share dimensions and kind")
    _native.layer_chain([l.data for l in layers], [l.mask for l in layers], [None] + list(ops),
                        out.data, out.mask, lazy=lazy)
    return out


def layer_area(layer, surface):
    """Surface area covered by the layer: sum of the per-texel area over mask != 0 (float64)."""
    sums, _ = _native.layer_area(surface.area, [layer.mask])
    return float(sums[0])


def layers_area(layers, surface):
    """Areas (and texel counts) of many layers in one fused pass -> (sums, counts) numpy arrays."""
    return _native.layer_area(surface.area, [l.mask for l in layers])


def label_area(layer, surface):
    """Area per label value of a uint8 layer -> (area[256], texels[256])."""
    return _native.label_area(surface.area, layer.data, layer.mask)


def layer_stats(layer):
    """(count, sum, min, max) of the layer's data over its valid texels."""
    return _native.layer_stats(layer.data, layer.mask)


def layer_precision(layer_or_coverage_count, mesh_area):
    """precision = surface area / covered texel count."""
    n = layer_or_coverage_count
    return mesh_area / float(n)
