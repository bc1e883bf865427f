"""editing -- the stroke pipeline: TEA (``apply_stroke``), TPA
(``build_outline_mask`` / ``apply_padding``), the projection formulas, and the north-star
selection brushes (``select_sphere``, ``select_sphere_batch``, ``select_threshold``).

Per stroke the host sends only scalars (the reference's "64 bytes"); planes, the
surface map and the depth map stay resident in HBM.
"""
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import DegenerateCamera, LayerMeshMismatch, StaleDepth, TargetMismatch

TRANSFER_BYTES_PER_STROKE = 64
DEFAULT_DEPTH_BIAS = 1e-4


@dataclass
class EditingTool:
    """SPEC.md:237-240."""
    px: float
    py: float
    shape: object                      # (T_h, T_w) bool/uint8 plane, numpy or CUDA tensor
    value: object = 1
    padding_radius: int = 1

    def __post_init__(self):
        if self.shape.ndim != 2 or self.shape.shape[0] < 1 or self.shape.shape[1] < 1:
            raise TargetMismatch("tool shape plane must be a non-empty 2-D plane")
        if self.padding_radius < 0:
            raise TargetMismatch("padding radius must be >= 0")

    @property
    def size(self):
        return int(self.shape.shape[1]), int(self.shape.shape[0])       # (T_w, T_h)


@dataclass
class EditProjection:
    """S_f, T_f and the kernel's tool map s = sfx*xn + bx, t = sfy*yn + by."""
    scale: tuple
    translate: tuple

    @property
    def kernel_factors(self):
        # window x = (xn+1)/2*W ; s = (x - (T_px - T_w/2))/T_w = S_f.x*xn + (0.5 - T_f.x)
        return self.scale[0], self.scale[1], 0.5 - self.translate[0], 0.5 - self.translate[1]


def compute_tool_projection(camera, tool):
    """SPEC.md:259-267 / PAPER.md:160-171:
    S_f = (W_w/(2 T_w), W_h/(2 T_h)),  T_f = ((T_px - 0.5 W_w)/T_w, (T_py - 0.5 W_h)/T_h)."""
    tw, th = tool.size
    ww, wh = float(camera.width), float(camera.height)
    if ww < 1 or wh < 1 or tw < 1 or th < 1:
        raise DegenerateCamera("window and tool sizes must be >= 1")
    return EditProjection(scale=(ww / (2.0 * tw), wh / (2.0 * th)),
                          translate=((tool.px - 0.5 * ww) / tw, (tool.py - 0.5 * wh) / th))


def project_fragment(s, t, w):
    """reject w <= 0, divide, reject outside the closed [0,1]^2 (KN:174, 189)."""
    if not w > 0.0:
        return None
    u, v = s / w, t / w
    if not (0.0 <= u <= 1.0 and 0.0 <= v <= 1.0):
        return None
    return u, v


@dataclass
class EditResult:
    """SPEC.md:245-247.  Counts stay on the device until read (no sync on the stroke path).

    ``edited_mask`` is the stroke context's EditedAreaMask plane: ONE plane per context, reset
    and rewritten by the next stroke -- it describes this stroke only until then (clone it, or bit-pack it with
    ``_native.pack_mask``, to keep it).  Results of ``stroke_gesture`` other than the last carry ``None``: all
    strokes of a gesture are queued by one host call and only the last stroke's marks survive it.
    ``duration_ms``: device time of the stroke when it was run with ``timed=True`` (two CUDA events around the
    engine call, read lazily), else ``None`` -- the stroke path does not pay for events nobody reads."""
    edited_mask: object
    _counts: object = None
    padded: int = 0
    transfer_bytes: int = TRANSFER_BYTES_PER_STROKE
    _cache: dict = field(default_factory=dict)
    _padded: object = None
    _events: object = None

    @property
    def duration_ms(self):
        if self._events is None:
            return None
        if "ms" not in self._cache:
            self._events[1].synchronize()
            self._cache["ms"] = float(self._events[0].elapsed_time(self._events[1]))
        return self._cache["ms"]

    @property
    def padded_count(self):
        """Texels written by the padding pass of ``stroke``."""
        return self.padded if self._padded is None else int(self._padded.item())

    def _read(self):
        if "c" not in self._cache:
            self._cache["c"] = [int(v) for v in self._counts.tolist()]
        return self._cache["c"]

    @property
    def edited_count(self):
        return self._read()[0]

    @property
    def fragments(self):
        c = self._read()
        return c[1] if len(c) > 1 else None

    def edited_indices(self):
        return self.edited_mask.view(_native._torch().uint8).flatten().nonzero().flatten()


class StrokeContext:
    """Everything TEA needs that changes only with the camera or the mesh: device triangle uv
    (grid units), clip coordinates MVP*vertex per triangle, the depth map, the surface map and a
    per-stroke ``edited`` plane (SPEC.md:253-255 EditedAreaMask, reset before each stroke)."""

    HALO_ROWS = 4                       # spare rows of a slab's edited plane = the largest padding radius of the culled path

    def __init__(self, mesh, camera, depth, surface, device="cuda"):
        torch = _native.require_cuda()
        self.mesh, self.camera, self.depth, self.surface = mesh, camera, depth, surface
        self.device = device
        self.tri_xy = surface.tri_xy
        # EditedAreaMask plane.  On a row slab of a taller atlas it carries HALO_ROWS spare rows above and below:
        # the neighbours' border rows of a stroke are received straight into them (sharding.exchange_halo_into)
        self.edited_ext = None
        if surface.rows != surface.height:
            self.edited_ext = (torch.zeros((surface.rows + 2 * self.HALO_ROWS, surface.width), dtype=torch.uint8, device=device),
                               self.HALO_ROWS)
            self.edited = self.edited_ext[0][self.HALO_ROWS:self.HALO_ROWS + surface.rows]
        else:
            self.edited = torch.zeros((surface.rows, surface.width), dtype=torch.uint8, device=device)
        self.scratch = _native.tea_scratch(mesh.num_triangles, surface.rows * surface.width, device)
        self._cstruct = None              # (outline data_ptr, ml_stroke_ctx) of the one-call stroke path
        self.refresh_camera()
        # footprint culling state: two tile bitmaps (this stroke / previous stroke) and whether the
        # edited plane may hold marks outside the previous bitmap (then it is reset as a whole)
        nwords = _native.tea_tile_words(surface.width, surface.rows)
        self.tiles = [torch.zeros(nwords, dtype=torch.int32, device=device) for _ in range(2)] if nwords else None
        self.edited_fully_dirty = False
        self.stroke_tiles = None          # tile bitmap of the last culled stroke (footprint of ctx.edited)
        self.cur = 0                      # tile buffer the next culled stroke writes; the other one is "previous"

    def refresh_camera(self):
        """(Re)derive everything that depends on the camera: clip coordinates MVP * vertex per triangle and
        the per-triangle evaluation records; remembers which camera state they belong to."""
        torch = _native._torch()
        clip = self.camera.clip_coords(self.mesh.vertices)[self.mesh.triangles]     # (T,3,4) float64
        self.tri_clip = torch.from_numpy(np.ascontiguousarray(clip)).to(self.device)
        self.recs = _native.tea_prepare(self.tri_xy, self.tri_clip, self.device)    # per-triangle evaluation records
        self.camera_key = self.camera.state_key()
        self._cstruct = None              # the one-call stroke struct holds pointers to tri_clip / recs

    def begin_culled_stroke(self):
        """Footprint-culled strokes clear the edited plane per footprint; after a whole-plane stroke
        the plane and the "previous" tile buffer are reset once."""
        if self.edited_fully_dirty:
            self.edited.zero_()
            self.tiles[self.cur ^ 1].zero_()
            self.edited_fully_dirty = False

    def end_culled_stroke(self):
        self.stroke_tiles = self.tiles[self.cur]      # footprint of the marks now in ctx.edited (for TPA)
        self.cur ^= 1                                  # this stroke's footprint is the next one's "previous"


def _stroke_checks(ctx, layer):
    s = ctx.surface
    key = ctx.camera.state_key()
    dkey = getattr(ctx.depth, "camera_key", None)
    if ctx.depth.generation != ctx.camera.generation or (dkey is not None and dkey != key):
        raise StaleDepth("depth map was rendered for camera generation %d, camera is at %d"
                         % (ctx.depth.generation, ctx.camera.generation))
    if ctx.camera_key != key:
        # the camera moved and the caller supplied a fresh depth map: the projected triangles and the
        # evaluation records of the context still belong to the old MVP -- rebuild them before any stroke
        ctx.refresh_camera()
    if layer.shape != (s.rows, s.width):
        raise TargetMismatch("layer is %s, surface map slab is %s" % (layer.shape, (s.rows, s.width)))
    if s.covered == 0 and s.row0 == 0 and s.rows == s.height:
        raise LayerMeshMismatch("no uv coverage at layer resolution")


def apply_stroke(ctx, tool, layer, *, eps=DEFAULT_DEPTH_BIAS, force_direct=False, cull=True, counts=None):
    """SPEC.md:277-285 TEA.  Uses the per-texel kernel over the cached triangle-id map when the uv
    layout has no overlaps (bit-identical), else the direct per-triangle kernel.
    ``cull`` (default) restricts the per-texel kernel to the stroke's footprint tiles, so a stroke
    costs O(triangles + footprint) instead of O(atlas); results are identical.  ``counts``: a
    ZEROED int64 device tensor of 2 elements to accumulate (edited, fragments) into (callers that queue many
    strokes keep one counter block per step instead of one allocation + fill per stroke)."""
    torch = _native._torch()
    _stroke_checks(ctx, layer)
    s = ctx.surface
    sfx, sfy, bx, by = compute_tool_projection(ctx.camera, tool).kernel_factors
    if counts is None:
        counts = torch.zeros(2, dtype=torch.int64, device=ctx.device)
    shape = tool.shape if _native._is_cuda_tensor(tool.shape) else _native._as_dev_bytes(tool.shape, ctx.device)
    args = (float(ctx.camera.width), float(ctx.camera.height), ctx.depth.plane, eps, sfx, sfy, bx, by,
            shape, layer.data, layer.mask, ctx.edited, tool.value)
    if s.overlap == 0 and not force_direct and ctx.tiles is not None and cull:
        # footprint-culled path: the EditedAreaMask reset is done inside the kernel
        # for the tiles the previous stroke could touch
        ctx.begin_culled_stroke()
        _native.tea_texels(ctx.tri_xy, ctx.tri_clip, s.tri_id, *args, row0=s.row0, counts=counts,
                           scratch=ctx.scratch, height=s.height, tiles=(ctx.tiles[ctx.cur], ctx.tiles[ctx.cur ^ 1]),
                           known_fragments=s.covered, recs=ctx.recs)
        ctx.end_culled_stroke()
    elif s.overlap == 0 and not force_direct:
        # whole-atlas form: the EditedAreaMask reset is folded into the id stream
        ctx.edited_fully_dirty = True
        ctx.stroke_tiles = None
        _native.tea_texels(ctx.tri_xy, ctx.tri_clip, s.tri_id, *args, row0=s.row0, counts=counts,
                           scratch=ctx.scratch, recs=ctx.recs, reset_edited=True, known_fragments=s.covered)
    else:
        ctx.edited.zero_()
        ctx.edited_fully_dirty = True
        ctx.stroke_tiles = None
        _native.raster_tea(ctx.tri_xy, ctx.tri_clip, *args, height=s.height, row0=s.row0, counts=counts)
    return EditResult(edited_mask=ctx.edited, _counts=counts)


def _timed(fn, timed):
    """Run fn() between two CUDA events when ``timed``; returns (result, events or None)."""
    if not timed:
        return fn(), None
    torch = _native._torch()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = fn()
    e1.record()
    return res, (e0, e1)


def stroke(ctx, tool, layer, outline, *, eps=DEFAULT_DEPTH_BIAS, cull=True, halo=None, timed=False):
    """The service's ``stroke`` (the edit the paper times): TEA followed by TPA with
    the tool's padding radius (details: ``_stroke``).  ``timed=True`` brackets the edit with two CUDA events;
    ``EditResult.duration_ms`` then reports its device time."""
    res, ev = _timed(lambda: _stroke(ctx, tool, layer, outline, eps=eps, cull=cull, halo=halo), timed)
    res._events = ev
    return res


def _stroke(ctx, tool, layer, outline, *, eps=DEFAULT_DEPTH_BIAS, cull=True, halo=None):
    """The service's ``stroke`` (the edit the paper times): TEA
    (``apply_stroke``) followed by TPA (``apply_padding``) with the tool's padding radius.
    ``outline`` is the layer-resolution outline mask (``build_outline_mask``).  The padded count
    stays on the device like the other counters (``EditResult.padded_count``).  With ``cull`` both
    passes touch only the stroke's footprint tiles.

    Row-sharded atlases (the context's surface map is a slab of a taller atlas): the padding stencil
    needs the neighbours' ``edited`` rows at the slab borders, so every rank calls ``stroke`` for
    every stroke and the ``radius`` border rows are exchanged point-to-point
    (``sharding.exchange_halo``; ``halo`` replaces that exchange, e.g. in single-process tests).  The
    padding pass then streams the slab's outline plane instead of walking footprint tiles."""
    torch = _native._torch()
    radius = tool.padding_radius
    s = ctx.surface
    as_u8 = outline.view(torch.uint8) if outline.dtype == torch.bool else outline
    one_call = (cull and ctx.tiles is not None and s.overlap == 0 and s.rows == s.height and 0 < radius <= 4
                and all(t.data_ptr() % 16 == 0 for t in (layer.data, layer.mask, as_u8)))
    if one_call:
        # the whole edit in ONE C call (ml_stroke: classify + TEA + TPA); counters stay on the device
        _stroke_checks(ctx, layer)
        ctx.begin_culled_stroke()
        if ctx._cstruct is None or ctx._cstruct[0] != as_u8.data_ptr():
            ctx._cstruct = (as_u8.data_ptr(), _native.stroke_ctx(
                ctx.tri_xy, ctx.tri_clip, ctx.recs, s.tri_id, ctx.scratch[0], ctx.scratch[1], ctx.tiles, ctx.edited, as_u8,
                width=s.width, height=s.height, row0=s.row0, rows=s.rows, known_fragments=s.covered))
        sfx, sfy, bx, by = compute_tool_projection(ctx.camera, tool).kernel_factors
        counts = torch.empty(3, dtype=torch.int64, device=ctx.device)
        _native.stroke_call(ctx._cstruct[1], ctx.cur, float(ctx.camera.width), float(ctx.camera.height), ctx.depth.plane,
                            eps, sfx, sfy, bx, by, tool.shape, layer.data, layer.mask, tool.value, radius, counts)
        ctx.end_culled_stroke()
        return EditResult(edited_mask=ctx.edited, _counts=counts[:2], _padded=counts[2:])
    res = apply_stroke(ctx, tool, layer, eps=eps, cull=cull)
    if radius > 0:
        pc = torch.zeros(1, dtype=torch.int64, device=ctx.device)
        if s.rows == s.height:
            _native.apply_padding(as_u8, ctx.edited, radius, layer.data, layer.mask, tool.value, counts=pc,
                                  tiles=ctx.stroke_tiles if cull else None)
        else:
            pad_slab(as_u8, ctx.edited, radius, layer.data, layer.mask, tool.value, pc, row0=s.row0, height=s.height,
                     tiles=ctx.stroke_tiles if cull else None, halo=halo, ext=ctx.edited_ext)
        res._padded = pc
    return res


def pad_slab(outline, edited, radius, data, mask, value, counts, *, row0, height, tiles=None, halo=None, ext=None):
    """TPA on one row slab of a taller atlas.  The ``radius`` rows next to a slab border need the
    neighbour's ``edited`` rows: they are exchanged point-to-point (``sharding.exchange_halo``, 16 KB per
    neighbour at 16384 texels; ``halo`` replaces the exchange in single-process tests and returns either
    ``(rows_above, rows_below)`` or an extended plane ``(ext, ext_row0)``) and those few border rows are
    padded by the streaming kernel over a 3 x radius-row window; the interior rows -- whose stencil never
    leaves the slab -- keep the footprint-culled tile pass.  Every output row is visited by exactly one of
    the passes, so planes and count equal the whole-plane result."""
    torch = _native._torch()
    rows, w = edited.shape
    if halo is None and ext is not None and radius <= ext[1]:
        # ``ext = (buf, margin)``: `edited` is buf[margin:margin + rows]; the halo rows land in buf's spare rows and
        # every window below is a VIEW of buf -- no concatenation, no allocation on the stroke path
        from . import sharding
        buf, margin = ext
        up_n, dn_n = sharding.exchange_halo_into(buf, margin, rows, row0, height, radius)
        top = min(radius, rows) if up_n else 0
        bot = min(radius, rows - top) if dn_n else 0
        culled = (tiles is not None and w % 128 == 0 and 0 < radius <= 4 and rows >= 2 * radius
                  and all(t.data_ptr() % 16 == 0 for t in (outline, edited, data, mask)))
        if not culled:
            _native.apply_padding(outline, buf[margin - up_n:margin + rows + dn_n], radius, data, mask, value, counts=counts,
                                  in_row0=row0 - up_n, out_row0=row0)
            return
        _native.apply_padding(outline, edited, radius, data, mask, value, counts=counts, tiles=tiles,
                              row_range=(top, rows - bot))
        if top:      # output rows [0, top): stencil rows [-radius, top + radius)
            _native.apply_padding(outline[:top], buf[margin - up_n:margin + min(rows, top + radius)], radius, data[:top],
                                  mask[:top], value, counts=counts, in_row0=row0 - up_n, out_row0=row0)
        if bot:      # output rows [rows - bot, rows)
            lo = max(0, rows - bot - radius)
            _native.apply_padding(outline[rows - bot:], buf[margin + lo:margin + rows + dn_n], radius, data[rows - bot:],
                                  mask[rows - bot:], value, counts=counts, in_row0=row0 + lo, out_row0=row0 + rows - bot)
        return
    if halo is None:
        from . import sharding
        up, dn = sharding.exchange_halo(edited, row0, height, radius, parts=True)
    else:
        got = halo(edited, row0, height, radius)
        if not (got[1] is None or torch.is_tensor(got[1])):              # (ext, ext_row0) form
            ext, ext_row0 = got
            k = row0 - ext_row0
            up = ext[:k] if k > 0 else None
            dn = ext[k + rows:] if ext.shape[0] > k + rows else None
        else:
            up, dn = got
    top = min(radius, rows) if up is not None and up.shape[0] else 0
    bot = min(radius, rows - top) if dn is not None and dn.shape[0] else 0
    culled = (tiles is not None and w % 128 == 0 and 0 < radius <= 4 and rows >= 2 * radius
              and all(t.data_ptr() % 16 == 0 for t in (outline, edited, data, mask)))
    if not culled:
        # no tile list: one streaming pass over the slab with the halo rows attached
        pieces = [p for p in (up, edited, dn) if p is not None and p.shape[0]]
        ext = torch.cat(pieces, 0) if len(pieces) > 1 else edited
        _native.apply_padding(outline, ext, radius, data, mask, value, counts=counts,
                              in_row0=row0 - (up.shape[0] if up is not None else 0), out_row0=row0)
        return
    _native.apply_padding(outline, edited, radius, data, mask, value, counts=counts, tiles=tiles,
                          row_range=(top, rows - bot))
    if top:      # output rows [0, top): stencil rows [-radius, top + radius)
        win = torch.cat([up, edited[:min(rows, top + radius)]], 0)
        _native.apply_padding(outline[:top], win, radius, data[:top], mask[:top], value, counts=counts,
                              in_row0=row0 - up.shape[0], out_row0=row0)
    if bot:      # output rows [rows - bot, rows)
        lo = max(0, rows - bot - radius)
        win = torch.cat([edited[lo:], dn], 0)
        _native.apply_padding(outline[rows - bot:], win, radius, data[rows - bot:], mask[rows - bot:], value,
                              counts=counts, in_row0=row0 + lo, out_row0=row0 + rows - bot)


def stroke_gesture(ctx, tools, layer, outline, *, eps=DEFAULT_DEPTH_BIAS):
    """A drag gesture (every pointer sample is one stroke): the strokes of ``tools`` are
    applied in order to ``layer`` -- same planes and counts as calling ``stroke`` for each -- but queued
    with ONE host call (``ml_stroke_sequence``), so the per-stroke cost is the device work, not the
    host's issue latency.  All tools share the padding radius.  Returns one ``EditResult`` per stroke
    (lazy device counters).  Contexts that cannot take the one-call path (slabs, overlapping uv
    layouts, radius 0 or > 4) fall back to a loop over ``stroke``."""
    torch = _native._torch()
    tools = list(tools)
    if not tools:
        return []
    s = ctx.surface
    radius = tools[0].padding_radius
    as_u8 = outline.view(torch.uint8) if outline.dtype == torch.bool else outline
    one_call = (ctx.tiles is not None and s.overlap == 0 and s.rows == s.height and 0 < radius <= 4
                and all(t.padding_radius == radius for t in tools)
                and all(t.data_ptr() % 16 == 0 for t in (layer.data, layer.mask, as_u8)))
    if not one_call:
        res = [stroke(ctx, t, layer, outline, eps=eps) for t in tools]
        for r in res[:-1]:
            r.edited_mask = None              # the shared EditedAreaMask plane now holds the last stroke's marks
        return res
    _stroke_checks(ctx, layer)
    ctx.begin_culled_stroke()
    if ctx._cstruct is None or ctx._cstruct[0] != as_u8.data_ptr():
        ctx._cstruct = (as_u8.data_ptr(), _native.stroke_ctx(
            ctx.tri_xy, ctx.tri_clip, ctx.recs, s.tri_id, ctx.scratch[0], ctx.scratch[1], ctx.tiles, ctx.edited, as_u8,
            width=s.width, height=s.height, row0=s.row0, rows=s.rows, known_fragments=s.covered))
    maps = [compute_tool_projection(ctx.camera, t).kernel_factors for t in tools]
    counts = torch.empty((len(tools), 3), dtype=torch.int64, device=ctx.device)
    _native.stroke_sequence_call(ctx._cstruct[1], ctx.cur, float(ctx.camera.width), float(ctx.camera.height),
                                 ctx.depth.plane, eps, maps, [t.shape for t in tools], layer.data, layer.mask,
                                 [t.value for t in tools], radius, counts)
    for _ in tools:
        ctx.end_culled_stroke()
    last = len(tools) - 1
    return [EditResult(edited_mask=ctx.edited if k == last else None, _counts=counts[k, :2], _padded=counts[k, 2:])
            for k in range(len(tools))]


# --------------------------------------------------------------------------------------------
# north-star selection brushes

def select_sphere(surface, layer, center, radius, value, edited=None, *, cull=True, counts=None):
    """Sphere brush: every covered texel whose surface point lies within ``radius`` of ``center``
    gets data = value, mask = true (definition: oracle ext_select_sphere).  ``cull`` (default) reads
    only the position-map tiles the sphere can reach (identical result, O(footprint) traffic);
    ``cull=False`` streams the whole map (12 B/texel)."""
    torch = _native._torch()
    if layer.shape != (surface.rows, surface.width):
        raise TargetMismatch("layer does not match the surface map")
    if edited is None:
        edited = torch.zeros(layer.shape, dtype=torch.uint8, device=surface.pos.device)
    if counts is None:
        counts = torch.zeros(1, dtype=torch.int64, device=surface.pos.device)
    _native.select_sphere(surface.pos, center, radius, layer.data, layer.mask, edited, value, counts=counts,
                          tiles=surface.tiles if cull else None)
    return EditResult(edited_mask=edited, _counts=counts, transfer_bytes=40)


def select_sphere_batch(surface, batch, *, cull=True):
    """K strokes over L layers in one pass (``batch`` = _native.StrokeBatch after upload); ``cull``
    as in ``select_sphere``."""
    _native.select_sphere_batch(surface.pos, batch, tiles=surface.tiles if cull else None)
    return batch.counts


def select_threshold(attr, valid, lo, hi, layer, value, edited=None, *, tiles=None, counts=None):
    """Attribute-threshold selection into ``layer`` (definition: oracle ext_select_threshold).
    ``tiles`` = ``_native.attr_tiles(attr)`` of a float32 attribute plane that does not change between
    selections (e.g. the surface map's height plane): only tiles whose value range meets [lo, hi]
    are read (identical result)."""
    torch = _native._torch()
    if tuple(attr.shape) != layer.shape:
        raise TargetMismatch("attribute plane does not match the layer")
    if edited is None:
        edited = torch.zeros(layer.shape, dtype=torch.uint8, device=attr.device)
    if counts is None:
        counts = torch.zeros(1, dtype=torch.int64, device=attr.device)
    _native.select_threshold(attr, valid, lo, hi, layer.data, layer.mask, edited, value, counts=counts, tiles=tiles)
    return EditResult(edited_mask=edited, _counts=counts, transfer_bytes=24)


# --------------------------------------------------------------------------------------------
# TPA

def build_outline_mask(mesh_or_coverage, resolution=None, thickness=1, device="cuda"):
    """(1) uv_coverage, (2) uncovered texels within Chebyshev distance
    ``thickness`` of a covered one."""
    torch = _native._torch()
    if thickness < 1:
        raise TargetMismatch("outline thickness must be >= 1")
    if _native._is_cuda_tensor(mesh_or_coverage):
        cov = mesh_or_coverage
    else:
        from .mesh_core import uv_coverage
        cov = uv_coverage(mesh_or_coverage, resolution, device=device)
    return _native.outline_mask(cov.view(torch.uint8) if cov.dtype == torch.bool else cov, thickness).view(torch.bool)


def apply_padding(layer, outline, edited, tool_or_value, radius=None):
    """outline texels within ``radius`` (Chebyshev) of an edited texel receive
    the stroke value.  Returns the padded texel count."""
    torch = _native._torch()
    value = tool_or_value.value if isinstance(tool_or_value, EditingTool) else tool_or_value
    if radius is None:
        radius = tool_or_value.padding_radius if isinstance(tool_or_value, EditingTool) else 1
    if tuple(outline.shape) != layer.shape or tuple(edited.shape) != layer.shape:
        raise TargetMismatch("grids must share the layer resolution")
    if radius <= 0:
        return 0
    as_u8 = lambda t: t.view(torch.uint8) if t.dtype == torch.bool else t
    return _native.apply_padding(as_u8(outline), as_u8(edited), radius, layer.data, layer.mask, value)
