"""bench module: plan invariants, frozen CSV schema, and on
the GPU the texture-engine parts of acceptance #5 (64 bytes/stroke), #6 (radius trend), #8
(precision of the flat square) and #11 (memory budget -> missing data point)."""
import numpy as np
import pytest

import paper_2501_14807_b200 as ml
from paper_2501_14807_b200 import bench, synth

GOLDEN_HEADER = "mesh,engine,level,radius,rep,time_ms,cells,transfer_bytes,build_ms,peak_bytes\n"


# ------------------------------------------------------------------ CPU: plan + CSV

def test_plan_defaults_and_invariants():
    p = bench.BenchPlan(meshes=["square"])
    assert p.resolutions == (2048, 4096, 8192) and p.depths == (11, 12, 13)
    assert p.radii == (10, 40, 70, 100, 200) and p.repetitions == 3
    with pytest.raises(ml.BadRequest):
        bench.BenchPlan(meshes=["square"], repetitions=2)
    with pytest.raises(ml.BadRequest):
        bench.BenchPlan(meshes=["square"], radii=(40, 10))
    with pytest.raises(ml.BadRequest):
        bench.BenchPlan(meshes=["square"], engine="voxels")
    with pytest.raises(ml.BadRequest):
        bench.BenchPlan(meshes=["square"], engine="octree", depths=(11,))


def test_plan_json():
    p = bench.BenchPlan.from_json('{"meshes": ["terrain:32"], "resolutions": [256], "radii": [5, 9], "repetitions": 4}')
    assert p.meshes == ("terrain:32",) and p.levels == (256,) and p.radii == (5, 9) and p.repetitions == 4
    for bad in ("{", "[]", '{"resolutions": [256]}', '{"meshes": [], "bogus": 1}'):
        with pytest.raises(ml.BadRequest):
            bench.BenchPlan.from_json(bad)


def test_csv_schema_golden():
    assert bench.csv_text([]) == GOLDEN_HEADER                                       # SPEC.md:521 empty plan
    r = bench.BenchRecord("square", "texture", 2048, 10, times_ms=[1.5, 1.25, 1.75], cells=42,
                          transfer_bytes=64, build_ms=3.0, peak_bytes=1000)
    missing = bench.BenchRecord("square", "texture", 8192, 10, outcome="memory_budget_exceeded")
    text = bench.csv_text([r, missing])
    assert text == (GOLDEN_HEADER +
                    "square,texture,2048,10,0,1.500000,42,64,3.000000,1000\n"
                    "square,texture,2048,10,1,1.250000,42,64,3.000000,1000\n"
                    "square,texture,2048,10,2,1.750000,42,64,3.000000,1000\n")
    assert (r.median_ms, r.min_ms, r.max_ms) == (1.5, 1.25, 1.75)
    assert missing.median_ms is None and list(missing.rows()) == []


def test_transfer_report_is_64_bytes_everywhere():
    plan = bench.BenchPlan(meshes=["sphere:2", "terrain:8", "square"])
    recs = bench.run_transfer_report(plan)
    assert len(recs) == 3 * 3 * 5 and {r.transfer_bytes for r in recs} == {64}


def test_octree_engine_has_no_cpu_fallback():
    """The octree baseline runs on the CUDA kernels like everything else: without a device it raises."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    plan = bench.BenchPlan(meshes=["square"], engine="octree", resolutions=(64,), depths=(2,))
    with pytest.raises(ml.BackendUnavailable):
        bench.run_transfer_report(plan)
    with pytest.raises(ml.BackendUnavailable):
        bench.run_radius_sweep(plan)


def test_stroke_input_hash_depends_on_every_input():
    cam = bench.make_camera("terrain:8", (64, 64))
    t1 = ml.EditingTool(px=32.0, py=32.0, shape=synth.circle_shape(5), value=7)
    t2 = ml.EditingTool(px=32.0, py=32.0, shape=synth.circle_shape(5), value=7)
    assert bench.stroke_input_hash(cam, t1) == bench.stroke_input_hash(cam, t2)
    t2.px = 33.0
    assert bench.stroke_input_hash(cam, t1) != bench.stroke_input_hash(cam, t2)
    cam2 = bench.make_camera("terrain:8", (64, 65))
    assert bench.stroke_input_hash(cam, t1) != bench.stroke_input_hash(cam2, t1)
    t3 = ml.EditingTool(px=32.0, py=32.0, shape=synth.circle_shape(6), value=7)
    assert bench.stroke_input_hash(cam, t1) != bench.stroke_input_hash(cam, t3)


def test_flat_square_mesh_area():
    assert ml.mesh_surface_area(synth.flat_square_mesh()) == 1.0
    assert ml.mesh_surface_area(synth.flat_square_mesh(2.0)) == 4.0


# ------------------------------------------------------------------ GPU

@pytest.mark.gpu
def test_precision_table_flat_square():
    """Acceptance #8, texture side: 1 m^2 square, 2048 texture -> 1e4/2048^2 cm^2."""
    plan = bench.BenchPlan(meshes=["square"], resolutions=(512, 2048))
    rows = bench.run_precision_table(plan)
    for row in rows:
        n = row["level"]
        assert row["covered"] == n * n
        assert abs(row["precision_cm2"] - 1e4 / (n * n)) <= 1e-9 * (1e4 / (n * n))
    assert rows[1]["precision_cm2"] < rows[0]["precision_cm2"]


@pytest.mark.gpu
def test_radius_sweep_small_plan(tmp_path):
    plan = bench.BenchPlan(meshes=["terrain:64", "sphere:3"], resolutions=(512,), radii=(4, 16, 40),
                           repetitions=3, window=(256, 256))
    recs = bench.run_radius_sweep(plan)
    assert [(r.mesh, r.level, r.radius) for r in recs] == [(m, 512, r) for m in plan.meshes for r in plan.radii]
    for r in recs:
        assert len(r.times_ms) == 3 and r.transfer_bytes == 64 and r.cells > 0 and r.build_ms > 0
    # a larger tool edits more cells on the same mesh
    assert recs[0].cells < recs[1].cells < recs[2].cells
    # same strokes without footprint culling: identical edited-cell counts
    flat = bench.run_radius_sweep(plan, cull=False)
    assert [r.cells for r in flat] == [r.cells for r in recs]
    out = tmp_path / "r.csv"
    bench.write_csv(recs, str(out))
    lines = out.read_text().splitlines()
    assert lines[0] + "\n" == GOLDEN_HEADER and len(lines) == 1 + len(recs) * 3


@pytest.mark.gpu
def test_radius_trend_fig5():
    """Acceptance #6, texture engine on the procedural terrain at 4096: median stroke
    time at r=200 over r=10 stays <= 2.  With footprint culling the small tool is the cheaper
    one (every point is below the whole-atlas curve); the whole-atlas path (cull=False) is the
    reference's flat curve and must satisfy the bound as well."""
    plan = bench.BenchPlan(meshes=["terrain:256"], resolutions=(4096,), radii=(10, 200), repetitions=5)
    flat = bench.run_radius_sweep(plan, cull=False)
    assert flat[1].median_ms / flat[0].median_ms <= 2.0
    culled = bench.run_radius_sweep(plan)
    assert culled[1].median_ms <= flat[1].median_ms * 1.5
    assert [r.cells for r in culled] == [r.cells for r in flat]


@pytest.mark.gpu
def test_memory_budget_records_missing_point():
    """Acceptance #11, texture side: a level over the budget is a missing data point,
    the level under it completes."""
    plan = bench.BenchPlan(meshes=["terrain:16"], resolutions=(256, 1024), radii=(8,),
                           budget_bytes=bench.texture_structure_bytes(512))
    recs = bench.run_radius_sweep(plan)
    assert recs[0].outcome == "ok" and len(recs[0].times_ms) == 3
    assert recs[1].outcome == "memory_budget_exceeded" and recs[1].times_ms == []
    assert bench.csv_text(recs).count("\n") == 1 + 3
