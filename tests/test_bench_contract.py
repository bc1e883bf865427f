"""bench.py --impl reference runs on the CPU (the oracle's C restatement with OpenMP): smoke-run it at a
tiny size and check the JSON contract of the line the driver parses (keys, types, the e2e and
cpu_baseline objects); ranks other than 0 print nothing."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["--impl", "reference", "--steps", "2", "--warmup", "1", "--atlas", "256", "--cpu-rows", "64", "--quads", "24",
        "--window", "96", "--layers", "4"]


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + ARGS, capture_output=True, text=True, env=env,
                          timeout=600)


def test_reference_arm_json_contract():
    r = _run({})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "Gtexel/s" and d["higher_is_better"] is True
    assert d["metric"].startswith("brush-apply + layer-op") and d["scaling"] == "weak" and d["vs_baseline"] is None
    assert d["steps"] == 2 and d["warmup"] == 1 and d["value"] > 0 and d["ms_per_step"] > 0
    assert d["data"] == "synthetic" and "workload" in d["config"] and d["config"]["layers"] == 4
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and "rows" in cb["sample"]
    assert set(cb["stage_ms"]) == {"tea", "tpa", "sphere", "batch", "chain", "mask_op", "threshold", "area"}
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_reference_arm_other_ranks_are_silent():
    r = _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0 and r.stdout.strip() == ""


import pytest


@pytest.mark.gpu
@pytest.mark.parametrize("extra", [[], ["--no-cull"]])
def test_gpu_arm_json_contract(extra):
    """bench.py (our arm) at a tiny atlas: one JSON line with every key of the contract."""
    args = ["--steps", "3", "--warmup", "3", "--atlas", "512", "--cpu-rows", "64", "--quads", "48", "--window", "128",
            "--layers", "4"] + extra
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["value"] > 0 and d["vs_baseline"] is None
    ro = d["roofline"]
    assert ro["bound"] == "hbm" and ro["unit"] == "GB/s" and ro["peak"] > 0 and abs(ro["frac"] - ro["achieved"] / ro["peak"]) < 1e-9
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["value"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["unit"] == d["unit"]
    per_step = 13 if not extra else 10
    assert d["gpu_launches"] == per_step * 3
    assert set(d["config"]["stage_results"]) == {"tea", "tpa", "sphere", "batch", "chain", "mask_op", "threshold", "area"}
    assert d["config"]["footprint_culling"] == (not extra)
    assert set(d["config"]["stream_kernels"]) == set(d["config"]["stage_results"]) | {"tea_id_stream_only"}
    assert set(d["config"]["stage_results_streamed"]) == set(d["config"]["stage_results"])
    assert d["value_streamed"] > 0 and d["ms_per_step_streamed"] > 0
    assert ro["streamed"]["bound"] == "hbm" and ro["streamed"]["kernel"] in d["config"]["stage_results"]
    # in-run parity of the two arms: GPU planes of the sampled rows == the CPU restatement's, both GPU paths
    pa = d["parity"]
    assert pa["checked"] is True and pa["ok"] is True, pa
    assert set(pa["paths"]) == {"default", "streamed"} and all(not v["mismatches"] for v in pa["paths"].values())
    assert pa["paths"]["default"]["planes_compared"] == 3 * 4 + 4
    # the reference's call shape with host planes
    hp = d["e2e_host_planes"]
    assert hp["ms_per_call"] > 0 and hp["equal_to_resident_stroke"] is True and hp["edited"] > 0
    assert hp["coverage_fill_ms_per_call"] > 0 and hp["coverage_fill_equals_surface_map"] is True
    assert hp["raster_depth_ms_per_call"] > 0 and hp["raster_depth_equals_resident"] is True


@pytest.mark.gpu
def test_gpu_arm_two_rank_rehearsal_over_gloo():
    """The N > 1 code path of bench.py (row slabs, stroke broadcast, halo exchange, area all-reduce, max over
    ranks) launched exactly like the driver does, with both ranks sharing cuda:0 through the gloo test hook
    (NCCL refuses two ranks on one device).  A rehearsal of the plumbing, not a measurement."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, ML_BENCH_BACKEND="gloo")
    args = ["--gpus", "2", "--steps", "3", "--warmup", "3", "--atlas", "512", "--cpu-rows", "64", "--quads", "48",
            "--window", "128", "--layers", "4"]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py")] + args,
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1                                            # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["parallelism"] == "row-sharded x2 (weak scaling)" and d["config"]["atlas"] == [1024, 512]
    assert d["cpu_baseline"] is None and d["parity"] is None          # N = 1 only
    # fused over peer memory (CUDA IPC between the two ranks on cuda:0); the all-gather form where IPC is not permitted
    assert d["config"]["area_reduce"].startswith("fused") or d["config"]["area_reduce"] == "all-gather"


@pytest.mark.gpu
def test_gpu_arm_config5_strong_scaling_rehearsal():
    """--config c5 (BASELINE config 5: 64 batched strokes + per-layer areas, strong scaling) at a tiny atlas, on one
    rank and on two gloo ranks sharing cuda:0: the rows are SPLIT over the ranks, the whole-job texel count stays."""
    import socket
    base = ["--config", "c5", "--steps", "3", "--warmup", "3", "--atlas", "512", "--cpu-rows", "64", "--quads", "48", "--layers", "4"]
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + base, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d1 = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d1["scaling"] == "strong" and d1["config"]["stages"] == ["batch", "area"] and d1["config"]["batch_strokes"] == 64
    assert d1["parity"]["ok"] is True and d1["config"]["atlas"] == [512, 512]
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, ML_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py")] + base + ["--gpus", "2"],
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d2 = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d2["n_gpus"] == 2 and d2["scaling"] == "strong" and d2["config"]["atlas"] == [512, 512]



@pytest.mark.gpu
def test_nccl_two_ranks_when_two_gpus_are_visible():
    """The real thing: two ranks, one GPU each, NCCL over NVLink (stroke-table broadcast, cross-rank area gather,
    halo rows point-to-point).  Runs whenever the box shows >= 2 GPUs, skips otherwise (the round's boxes have one)."""
    import socket
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    for cfg in ([], ["--config", "c5"]):
        args = cfg + ["--gpus", "2", "--steps", "5", "--warmup", "3", "--atlas", "1024", "--cpu-rows", "64", "--quads", "96",
                      "--window", "256", "--layers", "4"]
        r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py")] + args,
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
        assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
