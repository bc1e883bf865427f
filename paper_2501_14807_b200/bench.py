"""bench -- the reference's experiment harness for the stroke path: tool-radius
sweeps (Fig 5), transfer accounting (Fig 7) and the precision table (Table 1) for the TEXTURE
engine, emitted as CSV with the frozen column set of SPEC.md:549.

    python -m paper_2501_14807_b200.bench --plan plan.json --out results.csv

Plan JSON (every key optional except ``meshes``):
    {"meshes": ["sphere:5", "terrain:707", "square"],   # procedural stand-ins
     "engine": "texture",                                # or "octree" (levels = depths)
     "resolutions": [2048, 4096, 8192],                  # SPEC.md:505 defaults
     "depths": [11, 12, 13],                             # matched pairwise with resolutions
     "radii": [10, 40, 70, 100, 200],                    # px, Fig 5
     "repetitions": 3, "window": [1024, 1024], "units_to_cm": 100.0}

The timed call is ``editing.stroke`` (TEA + TPA, the edit the paper times), measured
with CUDA events around the engine call only, one warm-up discarded, medians over
the completed repetitions.  ``engine="octree"`` runs the OCT-TR baseline of
``octree.py`` (the paper's CPU competitor, here on the same GPU kernels' C ABI): its timed
call is ``octree_edit`` (``ml_tool_rays`` + ``raycast`` + leaf update), timed with the host clock
around a device synchronise because the edit has host work the events would not see.
"""
import csv
import hashlib
import io
import json
import statistics
from dataclasses import dataclass, field

import numpy as np

from . import _native, synth
from .errors import BadRequest, MemoryBudgetExceeded

#: SPEC.md:549 -- column set and order are frozen (golden-file test: tests/test_bench_csv.py)
CSV_COLUMNS = ("mesh", "engine", "level", "radius", "rep", "time_ms", "cells", "transfer_bytes",
               "build_ms", "peak_bytes")
DEFAULT_RESOLUTIONS = (2048, 4096, 8192)
DEFAULT_DEPTHS = (11, 12, 13)
DEFAULT_RADII = (10, 40, 70, 100, 200)


@dataclass
class BenchPlan:
    """SPEC.md:504-507.  Invariants: repetitions >= 3, radii sorted ascending, resolutions and
    depths matched pairwise."""
    meshes: tuple = ()
    engine: str = "texture"
    resolutions: tuple = DEFAULT_RESOLUTIONS
    depths: tuple = DEFAULT_DEPTHS
    radii: tuple = DEFAULT_RADII
    repetitions: int = 3
    window: tuple = (1024, 1024)
    units_to_cm: float = 100.0          # mesh units are metres unless declared otherwise
    budget_bytes: int = 0               # 0 = no budget; else MemoryBudgetExceeded -> missing data point

    def __post_init__(self):
        self.meshes = tuple(self.meshes)
        self.resolutions = tuple(int(r) for r in self.resolutions)
        self.depths = tuple(int(d) for d in self.depths)
        self.radii = tuple(self.radii)
        if self.engine not in ("texture", "octree"):
            raise BadRequest("engine must be 'texture' or 'octree'")
        if self.repetitions < 3:
            raise BadRequest("repetitions must be >= 3")
        if list(self.radii) != sorted(self.radii) or any(r <= 0 for r in self.radii):
            raise BadRequest("radii must be positive and sorted ascending")
        if self.engine == "octree" and len(self.depths) != len(self.resolutions):
            raise BadRequest("depths and resolutions are matched pairwise")
        if any(r < 1 for r in self.resolutions):
            raise BadRequest("resolutions must be >= 1")

    @classmethod
    def from_json(cls, text):
        try:
            d = json.loads(text)
        except ValueError as e:
            raise BadRequest("plan is not valid JSON: %s" % e)
        if not isinstance(d, dict) or "meshes" not in d:
            raise BadRequest("plan must be an object with a 'meshes' list")
        unknown = set(d) - set(cls.__dataclass_fields__)
        if unknown:
            raise BadRequest("unknown plan keys: %s" % sorted(unknown))
        return cls(**d)

    @property
    def levels(self):
        return self.resolutions if self.engine == "texture" else self.depths


@dataclass
class BenchRecord:
    """one (mesh, engine, level, radius) point.  ``times_ms`` holds the completed
    repetitions only; a missing data point (MemoryBudgetExceeded) has none."""
    mesh: str
    engine: str
    level: int
    radius: float
    times_ms: list = field(default_factory=list)
    cells: int = 0
    transfer_bytes: int = 0
    build_ms: float = 0.0
    peak_bytes: int = 0
    outcome: str = "ok"

    @property
    def median_ms(self):
        return statistics.median(self.times_ms) if self.times_ms else None

    @property
    def min_ms(self):
        return min(self.times_ms) if self.times_ms else None

    @property
    def max_ms(self):
        return max(self.times_ms) if self.times_ms else None

    def rows(self):
        """CSV rows: one per completed repetition (none for a missing data point)."""
        for rep, t in enumerate(self.times_ms):
            yield (self.mesh, self.engine, self.level, _num(self.radius), rep, "%.6f" % t, self.cells,
                   self.transfer_bytes, "%.6f" % self.build_ms, self.peak_bytes)


def _num(x):
    return int(x) if float(x).is_integer() else x


def write_csv(records, out):
    """Header row + one row per (record, repetition).  ``out`` is a path or a text stream; an empty
    record list gives the header row only."""
    own = isinstance(out, (str, bytes))
    f = open(out, "w", newline="") if own else out
    try:
        w = csv.writer(f, lineterminator="\n")
        w.writerow(CSV_COLUMNS)
        for r in records:
            for row in r.rows():
                w.writerow(row)
    finally:
        if own:
            f.close()


def csv_text(records):
    s = io.StringIO()
    write_csv(records, s)
    return s.getvalue()


# --------------------------------------------------------------------------------------------
# procedural meshes and the camera script (SPEC.md:544 desk-scale substitutes)

def make_mesh(spec):
    """'sphere:<level>' (icosphere, one island per triangle), 'terrain:<quads per side>' (bumpy
    heightfield, single island), 'square' (flat 1 x 1 unit square filling the whole atlas)."""
    name, _, arg = spec.partition(":")
    if name == "sphere":
        return synth.icosphere_mesh(int(arg or 5))
    if name == "terrain":
        return synth.heightfield_mesh(int(arg or 707), margin=0.01)
    if name == "square":
        return synth.flat_square_mesh()
    raise BadRequest("unknown mesh spec %r" % (spec,))


def make_camera(spec, window):
    """One fixed camera per mesh family, looking at the surface centre: identical for every
    engine / level / radius of a plan."""
    ww, wh = int(window[0]), int(window[1])
    if spec.partition(":")[0] == "sphere":
        return synth.default_camera(ww, wh)
    return synth.default_camera(ww, wh, eye=(0.5, 0.5, 1.6), target=(0.5, 0.5, 0.0), fovy=40.0, near=0.2, far=5.0)


def stroke_input_hash(camera, tool):
    """Hash of everything an engine receives for one stroke: camera state and tool parameters
    ("asserted by hashing the inputs")."""
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(camera.view, dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(camera.projection, dtype=np.float64).tobytes())
    h.update(np.array([camera.width, camera.height], dtype=np.int64).tobytes())
    h.update(np.array([tool.px, tool.py], dtype=np.float64).tobytes())
    shape = tool.shape.cpu().numpy() if _native._is_cuda_tensor(tool.shape) else np.asarray(tool.shape)
    h.update(np.array(shape.shape, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(shape).astype(np.uint8).tobytes())
    h.update(repr(tool.value).encode())
    return h.hexdigest()


def texture_structure_bytes(resolution, kind_bytes=1):
    """Bytes the texture engine keeps per layer resolution: layer data + mask, the edited-area and
    outline masks (1 B/texel each) and the surface map (id 4 + pos 12 + nrm 12 + area 4)."""
    return resolution * resolution * (kind_bytes + 1 + 1 + 1 + 32)


class _TextureSetup:
    """Everything the texture engine builds once per (mesh, resolution): surface map, depth map,
    outline mask, stroke context, one uint8 layer.  ``build_ms`` is the device time of the build."""

    def __init__(self, mesh, camera, resolution, budget_bytes=0):
        from . import editing, layer_core, mesh_core
        from .raster_device import TexturePool
        torch = _native.require_cuda()
        self.peak_bytes = texture_structure_bytes(resolution)
        if budget_bytes and self.peak_bytes > budget_bytes:
            raise MemoryBudgetExceeded("texture level %d needs %d bytes, budget is %d"
                                       % (resolution, self.peak_bytes, budget_bytes))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        self.surface = mesh_core.build_surface_map(mesh, resolution, resolution)
        self.depth = mesh_core.render_depth(mesh, camera)
        self.outline = editing.build_outline_mask(self.surface.coverage, thickness=1)
        b.record()
        torch.cuda.synchronize()
        self.build_ms = a.elapsed_time(b)
        self.ctx = editing.StrokeContext(mesh, camera, self.depth, self.surface)
        self.pool = TexturePool(budget_texels=4 * resolution * resolution)
        self.layer = layer_core.create_layer("bench", "uint8", resolution, resolution, pool=self.pool)


def _tool(camera, radius):
    from .editing import EditingTool
    return EditingTool(px=0.5 * camera.width, py=0.5 * camera.height, shape=synth.circle_shape(radius), value=7)


class _OctreeSetup:
    """What the octree engine builds once per (mesh, depth): the surface octree and one uint8 layer."""

    def __init__(self, mesh, depth, budget_bytes=0):
        from . import octree
        self.octree = octree.build_octree(mesh, depth, budget_bytes=budget_bytes)
        self.layer = octree.create_octree_layer(self.octree, "uint8")
        self.build_ms = self.octree.build_ms
        self.peak_bytes = self.octree.peak_bytes


def _octree_radius_sweep(plan):
    import time
    from . import octree
    torch = _native.require_cuda()
    records = []
    for spec in plan.meshes:
        mesh = make_mesh(spec)
        camera = make_camera(spec, plan.window)
        for level in plan.levels:
            try:
                setup = _OctreeSetup(mesh, level, plan.budget_bytes)
            except MemoryBudgetExceeded:
                torch.cuda.empty_cache()
                records += [BenchRecord(spec, plan.engine, level, r, outcome="memory_budget_exceeded")
                            for r in plan.radii]
                continue
            for radius in plan.radii:
                tool = _tool(camera, radius)
                tool.shape = _native._as_dev_bytes(tool.shape, "cuda")   # like the texture engine's sweep
                rec = BenchRecord(spec, plan.engine, level, radius, build_ms=setup.build_ms,
                                  peak_bytes=setup.peak_bytes)
                res = None
                for rep in range(plan.repetitions + 1):              # rep 0 = discarded warm-up
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    res = octree.octree_edit(setup.octree, setup.layer, mesh, camera, tool)
                    torch.cuda.synchronize()
                    if rep:
                        rec.times_ms.append((time.perf_counter() - t0) * 1e3)
                rec.cells = res.edited_count
                rec.transfer_bytes = res.transfer_bytes
                records.append(rec)
            del setup
            torch.cuda.empty_cache()
    return records


def run_radius_sweep(plan, cull=True):
    """one record per (mesh, level, radius); identical camera and stroke position
    for every point.  A level over the plan's memory budget is recorded as a missing data point."""
    from . import editing
    if plan.engine == "octree":
        return _octree_radius_sweep(plan)
    torch = _native.require_cuda()
    records = []
    for spec in plan.meshes:
        mesh = make_mesh(spec)
        camera = make_camera(spec, plan.window)
        for level in plan.levels:
            try:
                setup = _TextureSetup(mesh, camera, level, plan.budget_bytes)
            except MemoryBudgetExceeded:
                records += [BenchRecord(spec, plan.engine, level, r, outcome="memory_budget_exceeded")
                            for r in plan.radii]
                continue
            for radius in plan.radii:
                tool = _tool(camera, radius)
                tool.shape = _native._as_dev_bytes(tool.shape, "cuda")
                rec = BenchRecord(spec, plan.engine, level, radius, build_ms=setup.build_ms,
                                  peak_bytes=setup.peak_bytes)
                res = None
                for rep in range(plan.repetitions + 1):              # rep 0 = discarded warm-up
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    a.record()
                    if cull:
                        res = editing.stroke(setup.ctx, tool, setup.layer, setup.outline)
                    else:
                        res = editing.apply_stroke(setup.ctx, tool, setup.layer, cull=False)
                        editing.apply_padding(setup.layer, setup.outline, setup.ctx.edited, tool)
                    b.record()
                    torch.cuda.synchronize()
                    if rep:
                        rec.times_ms.append(a.elapsed_time(b))
                rec.cells = res.edited_count
                rec.transfer_bytes = res.transfer_bytes
                records.append(rec)
            del setup
            torch.cuda.empty_cache()
    return records


def run_transfer_report(plan):
    """CPU->GPU bytes per stroke; the texture engine moves the 64-byte matrix in
    every configuration."""
    from .editing import TRANSFER_BYTES_PER_STROKE
    if plan.engine == "octree":                                      # crossed leaves x 4
        from . import octree
        out = []
        for spec in plan.meshes:
            mesh = make_mesh(spec)
            for level in plan.levels:
                try:
                    tree = octree.build_octree(mesh, level, budget_bytes=plan.budget_bytes)
                except MemoryBudgetExceeded:
                    out += [BenchRecord(spec, plan.engine, level, r, outcome="memory_budget_exceeded")
                            for r in plan.radii]
                    continue
                out += [BenchRecord(spec, plan.engine, level, r, cells=tree.leaf_count,
                                    transfer_bytes=octree.octree_upload_size(tree), build_ms=tree.build_ms,
                                    peak_bytes=tree.peak_bytes) for r in plan.radii]
                del tree
        return out
    return [BenchRecord(spec, plan.engine, level, r, transfer_bytes=TRANSFER_BYTES_PER_STROKE)
            for spec in plan.meshes for level in plan.levels for r in plan.radii]


def run_precision_table(plan):
    """layer precision = surface area / covered texels, in cm^2.  Returns dicts
    {mesh, level, covered, area_cm2, precision_cm2}."""
    from . import layer_core, mesh_core
    _native.require_cuda()
    out = []
    for spec in plan.meshes:
        mesh = make_mesh(spec)
        area_cm2 = mesh_core.mesh_surface_area(mesh) * plan.units_to_cm ** 2
        for level in plan.levels:
            if plan.engine == "octree":                              # area / crossed leaves
                from . import octree
                tree = octree.build_octree(mesh, level, budget_bytes=plan.budget_bytes)
                out.append({"mesh": spec, "level": level, "covered": tree.leaf_count, "area_cm2": area_cm2,
                            "precision_cm2": octree.octree_precision(tree, mesh, plan.units_to_cm)})
                continue
            covered = int(mesh_core.uv_coverage(mesh, level).sum().item())
            out.append({"mesh": spec, "level": level, "covered": covered, "area_cm2": area_cm2,
                        "precision_cm2": layer_core.layer_precision(covered, area_cm2) if covered else None})
    return out


def main(argv=None):
    import argparse
    ap = argparse.ArgumentParser(prog="bench", description=__doc__.split("\n\n")[0])
    ap.add_argument("--plan", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--no-cull", action="store_true", help="time the whole-atlas TEA path (flat radius curve)")
    args = ap.parse_args(argv)
    with open(args.plan) as f:
        plan = BenchPlan.from_json(f.read())
    records = run_radius_sweep(plan, cull=not args.no_cull) if plan.meshes else []
    write_csv(records, args.out)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
