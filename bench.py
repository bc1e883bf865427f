#!/usr/bin/env python
"""bench.py -- brush-apply + layer-op throughput at a 16384^2 atlas (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3c4|c5]

One STEP = one pass of every hot-path stage over this rank's atlas slab.  Default workload
(``--config c3c4``): the C3+C4 workload of BASELINE.json -- a 16384 x 16384 slab (268.4 Mtexel) per
rank, 8 uint8 layers (``--layers 64`` gives C4), the 999,698-triangle heightfield mesh -- with the
stages, in the order of ``STAGES`` (streaming stages first):

    chain      fused layer-algebra chain ((L0 u L1) n L2) \\ L3 ... over 8 uint8 layers (C3)
    mask_op    binary union of two bare uint8 mask planes (the 3 B/texel streaming kernel)
    area       per-layer area of all L layers in one fused pass (+ cross-rank sum when N > 1)
    threshold  attribute-threshold selection on the float32 attribute plane pos.z (C3)
    tea        the paper's projective brush (TEA, KN:135-203) over the cached triangle-id map
    tpa        the paper's padding pass (TPA): outline texels next to the stroke
    sphere     one sphere-brush stroke over the float32x3 position map
    batch      K sphere strokes (one per layer) batched in ONE pass over the position map

metric = texel passes per second: (stages x slab texels x ranks) / step time, in Gtexel/s.  The run
measures it FOUR ways and prints all of them in one JSON line:

    value            the public API's default path, everything resident in HBM, CUDA events.  The brush /
                     selection stages are footprint-culled (a stroke reads only the tiles it can reach), the
                     chain reads a data vector only where the masks let it reach the result: these stages
                     skip most of their SURVEY 8(d) bytes BY DESIGN, so ``value`` counts nominal texel passes.
    value_streamed   the same steps with every stage forced to stream the whole atlas (``cull=False`` /
                     eager chain): the byte-honest figure; its stage table is the HBM-roofline evidence.
    e2e              the default path driven from HOST stroke records (pinned memory -> device every step)
                     with every stage's results (edit counts, areas) read back to the host every step.
    e2e_host_planes  the reference's own call shape: the drop-in twin ``raster_tea`` (KN:135-136) called
                     per step with numpy planes in pageable host memory, everything else of the call
                     (uploads, kernel, sparse write-back into the caller's planes) inside the timed region.

``roofline`` is quoted for the slowest stage of the default step (algorithmic AND measured-DRAM
fractions; DRAM bytes per launch from profiles/traffic.json, an ncu --set full capture), and
``roofline.streamed`` for the slowest stage of the streamed step.  ``stream_kernels`` re-times each
whole-atlas stage alone inside a CUDA graph (no host launch latency).

``parity`` (untimed): after the timed loops the GPU planes are reset, P steps are run on the default path
and again on the streamed path, and the reference-side CPU implementation (oracle/kn_port.c) runs the same
P steps on its row sample; every layer plane, edited plane, chain / mask_op result and per-layer area of the
sampled rows must agree (planes bit for bit, areas to 1e-10).  A mismatch makes the run exit non-zero.

Inputs are far larger than the 126 MB L2 (every plane is >= 268 MB), so no explicit L2 flush is
needed between iterations.

Multi-GPU (torchrun, one rank per GPU): weak scaling -- the atlas grows to 16384 x (16384*N) and
each rank owns one 16384-row slab; the only exchanges are the stroke-table broadcast, the TPA halo rows and
the cross-rank area sum, which is fused into the reduction kernel (system-scope atomics into every rank's
result row over IPC-mapped peer memory; ``ML_AREA_REDUCE=gather`` = one all-gather of 16 L bytes instead).  ``--config c5`` is BASELINE config 5: a
32768^2 atlas with the 9,999,392-triangle heightfield, STRONG scaling (the rows are split over the
ranks), stages batch (64 strokes) + area.

``--impl reference`` times the reference-side CPU implementation (oracle/kn_port.c, the C
restatement of the reference's numpy kernels, row-parallel over all host threads, per-band triangle
lists, fused chain / batch / areas) on a bounded row sample of the same workload.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# The long streaming stages come first: after the end-of-step read-back of the e2e loop the host queues
# them in a few microseconds and prepares the (host-heavier) brush calls while the GPU is busy.
STAGES = ("chain", "mask_op", "area", "threshold", "tea", "tpa", "sphere", "batch")
CHAIN_OPS = ["union", "intersection", "difference", "union", "masking", "difference", "union"]
BRUSH = ("tea", "tpa", "sphere", "batch", "threshold")
CONFIGS = {
    "c3c4": dict(atlas=16384, quads=707, layers=8, scaling="weak", stages=",".join(STAGES), batch=0),
    "c5": dict(atlas=32768, quads=2236, layers=8, scaling="strong", stages="batch,area", batch=64),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3c4", choices=sorted(CONFIGS))
    ap.add_argument("--atlas", type=int, default=None, help="atlas width (and per-rank slab height under weak scaling)")
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--quads", type=int, default=None, help="heightfield quads per side (707 -> 999,698 tris)")
    ap.add_argument("--window", type=int, default=1024)
    ap.add_argument("--cpu-rows", type=int, default=1024, help="rows of the slab the CPU baseline processes")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline / parity / host-plane legs")
    ap.add_argument("--no-cull", action="store_true",
                    help="the PRIMARY loops stream the whole atlas too (value == value_streamed)")
    ap.add_argument("--parity-steps", type=int, default=2)
    ap.add_argument("--host-plane-reps", type=int, default=8)
    ap.add_argument("--stages", default=None)
    ap.add_argument("--profile-loop", default=None, choices=["default", "streamed"],
                    help="ncu target: set-up, then ONLY the resident loop of that path (W warm-up + K timed steps), a short "
                         "JSON line with the stage times, exit -- so that a launch list holds the kernels of one path only")
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    for k in ("atlas", "layers", "quads", "stages"):
        if getattr(a, k) is None:
            setattr(a, k, cfg[k])
    a.scaling = cfg["scaling"]
    a.batch = cfg["batch"]
    return a


# ------------------------------------------------------------------------------------------------
# workload definition shared by both arms

class Workload:
    def __init__(self, args, world_size):
        from paper_2501_14807_b200 import synth
        self.A = args.atlas
        self.width = args.atlas
        strong = getattr(args, "scaling", "weak") == "strong"
        self.height = args.atlas if strong else args.atlas * world_size
        self.L = args.layers
        self.K = getattr(args, "batch", 0) or self.L               # strokes per batched pass
        self.mesh = synth.heightfield_mesh(args.quads, margin=0.01)   # 1% uv border: a real island outline for TPA
        self.cam = synth.default_camera(args.window, args.window, eye=(0.5, 0.5, 1.6), target=(0.5, 0.5, 0.0),
                                        fovy=40.0, near=0.2, far=5.0)
        self.tool_shape = synth.circle_shape(70)                     # the paper's mid radius (70 px)
        self.eps = 1e-4
        nchain = min(8, self.L)
        self.chain_n = nchain
        self.chain_ops = CHAIN_OPS[:nchain - 1]
        z = self.mesh.vertices[:, 2]
        self.thr = (float(np.percentile(z, 40.0)), float(np.percentile(z, 60.0)))   # C3 window
        # pre-painting (seeded): 4 strokes per layer
        self.seed_strokes, self.seed_labels = synth.sphere_strokes(self.mesh, 4 * self.L, seed=synth.SEED + 3,
                                                                   rmin_frac=0.02, rmax_frac=0.08)

    def step_inputs(self, i):
        """Per-step host inputs (seeded): tool position, one sphere stroke, K batch strokes."""
        from paper_2501_14807_b200 import synth
        rng = np.random.default_rng(synth.SEED + 100 + i)
        w = self.cam.width
        tool_xy = rng.uniform(0.3 * w, 0.7 * w, size=2)
        strokes, labels = synth.sphere_strokes(self.mesh, self.K + 1, seed=synth.SEED + 1000 + i,
                                               rmin_frac=0.01, rmax_frac=0.05)
        # the threshold selection re-labels its window with a different value every step (an identical selection
        # repeated would leave nothing to write from the second step on)
        return dict(tool_xy=tool_xy, sphere=strokes[0], sphere_value=int(labels[0]), thr_value=9 + (i % 7),
                    batch=strokes[1:], batch_layers=(np.arange(self.K) % self.L).astype(np.int32), batch_values=labels[1:])

    def algorithmic_bytes(self, n, stage, T, hits=0):
        """Algorithmic HBM bytes of one stage over n texels: the read stream plus,
        for the brushes, `hits` texels x (1 B edited read + 1 B edited + 1 B mask + 1 B uint8 data
        written).  tea additionally resets the 1 B/texel edited plane and reads the
        clip coordinates of every triangle once for the classification pass."""
        L = self.L
        base = {"tea": 4 * n + n + T * 12 * 8 + self.cam.width * self.cam.height * 4,
                "sphere": 12 * n, "batch": 12 * n,
                "chain": (self.chain_n + 1) * 2 * n, "mask_op": 3 * n,
                "tpa": n, "threshold": 4 * n, "area": (4 * -(-L // 8) + L) * n}[stage]
        return base + 4 * int(hits)


def sample_clocks(stop, out):
    """nvidia-smi clocks line of B200_PROFILING.md, one sample every 100 ms; every line is stamped with the
    host clock as it arrives so that the summary can keep the samples taken inside the timed regions."""
    q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    try:
        p = subprocess.Popen(["nvidia-smi", "--query-gpu=" + q, "--format=csv,noheader,nounits", "-lms", "100",
                              "-i", os.environ.get("LOCAL_RANK", "0")], stdout=subprocess.PIPE, text=True, bufsize=1)
    except OSError:
        return

    def reader():
        for line in p.stdout:
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                out.append((time.time(), f))

    rd = threading.Thread(target=reader, daemon=True)
    rd.start()
    stop.wait()
    p.terminate()
    rd.join(timeout=5)


def clocks_summary(samples, windows=()):
    """Median SM clock and throttle reasons of the samples taken inside the timed regions (``windows`` =
    [(t0, t1), ...] host times).  A timed region shorter than the sampling interval can hold no sample;
    the samples taken under the same load around it (warm-up .. end of the e2e loop) are used then."""
    if not samples:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
    inside = [f for t, f in samples if any(t0 <= t <= t1 + 0.05 for t0, t1 in windows)]
    scope = "timed regions"
    if len(inside) < 2:
        inside = [f for _, f in samples]
        scope = "warm-up + timed regions (timed regions shorter than the sampling interval)"
    sm = sorted(float(s[1]) for s in inside if s[1].replace(".", "").isdigit())
    reasons = set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for s in inside:
        for name, v in zip(names, s[5:9]):
            if v.lower().startswith("active"):
                reasons.add(name)
    return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": float(inside[0][2]),
            "reasons": sorted(reasons), "samples": len(inside), "scope": scope}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def time_graph(fn, inner=10, reps=7, warm=2):
    """Median ms per call of `fn` over `reps` replays of a CUDA graph holding `inner` back-to-back calls (a single
    call between two events on an idle GPU also measures the host's 10-30 us issue latency).  Falls back to
    eager back-to-back calls if the call cannot be captured.  Returns (ms, graphed)."""
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    graph = None
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(inner):
                fn()
        graph = g
    except Exception:            # not capturable (host sync inside): eager back-to-back launches
        torch.cuda.synchronize()
    ts = []
    for _ in range(reps + 1):
        a.record()
        if graph is not None:
            graph.replay()
        else:
            for _ in range(inner):
                fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / inner)
    return float(np.median(ts[1:])), graph is not None


# ------------------------------------------------------------------------------------------------
# CPU arm (reference / cpu_baseline / parity): oracle C restatement, all host threads, bounded row sample

class CpuArm:
    """The reference algorithm at its best on the host cores: row-parallel OpenMP over all threads, triangles
    pre-binned per row band (no re-scan of the triangle list per band), the chain, the stroke batch and the
    per-layer areas each as ONE fused pass (oracle/kn_port.c ext_*_fused / ext_layer_chain / ext_layers_area)."""

    def __init__(self, wl, rows):
        from oracle import kn
        self.kn, self.wl = kn, wl
        self.threads = kn.max_threads()
        self.rows = min(rows, wl.A)
        self.row0 = (wl.A - self.rows) // 2                      # a slab from the middle of rank 0's rows
        W = wl.width
        m = wl.mesh
        self.tri_xy = m.tri_uv_texels(wl.width, wl.height)
        self.tri_clip = wl.cam.clip_coords(m.vertices)[m.triangles]
        t0 = time.time()
        self.surf = kn.surface_map(self.tri_xy, m.tri_pos(), m.tri_nrm(), wl.width, wl.height,
                                   rows=(self.row0, self.row0 + self.rows), threads=self.threads)
        from paper_2501_14807_b200.mesh_core import window_triangles
        xy, zn = window_triangles(m, wl.cam)
        self.depth = np.ones((wl.cam.height, wl.cam.width), np.float32)
        kn.raster_depth(xy, zn, self.depth, threads=self.threads)
        self.setup_s = time.time() - t0
        n = self.rows * W
        self.n = n
        mk = lambda dt: [np.zeros((self.rows, W), dt) for _ in range(wl.L)]
        self.data, self.mask, self.edited = mk(np.uint8), mk(np.uint8), mk(np.uint8)
        self.tea_edited = np.zeros((self.rows, W), np.uint8)      # the stroke context's EditedAreaMask
        self.out_d, self.out_m = np.zeros((self.rows, W), np.uint8), np.zeros((self.rows, W), np.uint8)
        self.outline = kn.outline((self.surf["tri_id"] >= 0).astype(np.uint8), 1, threads=self.threads)
        self.tmp_m = np.zeros((self.rows, W), np.uint8)
        for k in range(len(wl.seed_strokes)):                     # same pre-painting as the GPU arm
            L = k % wl.L
            kn.select_sphere(self.surf["pos"], wl.seed_strokes[k, :3], wl.seed_strokes[k, 3], self.data[L],
                             self.mask[L], self.edited[L], wl.seed_labels[k], threads=self.threads)

    def step(self, i, stages):
        kn, wl, th = self.kn, self.wl, self.threads
        inp = wl.step_inputs(i)
        res = {}
        t = {}
        for st in stages:
            t0 = time.perf_counter()
            if st == "tea":
                from paper_2501_14807_b200 import EditingTool, compute_tool_projection
                tool = EditingTool(px=float(inp["tool_xy"][0]), py=float(inp["tool_xy"][1]), shape=wl.tool_shape, value=7)
                sfx, sfy, bx, by = compute_tool_projection(wl.cam, tool).kernel_factors
                self.tea_edited[:] = 0
                res["tea"] = kn.raster_tea_slab(self.tri_xy, self.tri_clip, float(wl.cam.width), float(wl.cam.height),
                                                self.depth, wl.eps, sfx, sfy, bx, by, wl.tool_shape, self.data[0],
                                                self.mask[0], self.tea_edited, 7, wl.height, self.row0, th)
            elif st == "tpa":
                res["tpa"] = kn.padding(self.outline, self.tea_edited, 1, self.data[0], self.mask[0], 7, threads=th)
            elif st == "sphere":
                s = inp["sphere"]
                res["sphere"] = kn.select_sphere(self.surf["pos"], s[:3], s[3], self.data[1 % wl.L], self.mask[1 % wl.L],
                                                 self.edited[1 % wl.L], inp["sphere_value"], threads=th)
            elif st == "batch":
                res["batch"] = kn.select_sphere_batch(self.surf["pos"], inp["batch"], inp["batch_layers"], inp["batch_values"],
                                                      self.data, self.mask, self.edited, threads=th)
            elif st == "chain":
                kn.layer_chain(wl.chain_ops, self.data[:wl.chain_n], self.mask[:wl.chain_n], self.out_d, self.out_m, threads=th)
            elif st == "mask_op":
                kn.layer_op("union", None, self.mask[0], None, self.mask[1 % wl.L], None, self.tmp_m, threads=th)
            elif st == "threshold":
                res["threshold"] = kn.select_threshold(self.surf["pos"][2], None, wl.thr[0], wl.thr[1], self.data[2 % wl.L],
                                                       self.mask[2 % wl.L], self.edited[2 % wl.L], inp["thr_value"], threads=th)
            elif st == "area":
                res["area"] = kn.layers_area(self.surf["area"], self.mask, threads=th)
            t[st] = time.perf_counter() - t0
        return t, res

    DESCRIPTION = ("oracle/kn_port.c (C restatement of the reference numpy kernels): OpenMP over row bands with per-band "
                   "triangle lists, fused chain / stroke batch / per-layer areas")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    stages = [s for s in args.stages.split(",") if s]
    wl = Workload(args, 1)
    arm = CpuArm(wl, args.cpu_rows)
    for i in range(args.warmup):
        arm.step(i, stages)
    t0 = time.perf_counter()
    per = {s: 0.0 for s in stages}
    for i in range(args.steps):
        t, _ = arm.step(args.warmup + i, stages)
        for s in stages:
            per[s] += t[s]
    el = time.perf_counter() - t0
    value = len(stages) * arm.n * args.steps / el / 1e9
    sample = "%d of %d rows of the %dx%d slab (%.1f Mtexel); %s" % (
        arm.rows, wl.A, wl.A, wl.width, arm.n / 1e6, CpuArm.DESCRIPTION)
    print(json.dumps({
        "impl": "reference", "metric": "brush-apply + layer-op texel passes per second at 16384^2 atlas",
        "value": value, "unit": "Gtexel/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f64 decisions on u8/u32/f32 planes", "data": "synthetic",
        "config": workload_config(args, wl, stages),
        "cpu_baseline": {"value": value, "unit": "Gtexel/s", "cores": arm.threads, "kind": "port", "sample": sample,
                         "stage_ms": {s: per[s] / args.steps * 1e3 for s in stages}},
        "e2e": {"value": value, "unit": "Gtexel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def workload_config(args, wl, stages):
    return {"workload": "%s: %dx%d atlas%s, %d uint8 layers, %d-triangle heightfield mesh; stages %s"
                        % ({"c3c4": "C3+C4", "c5": "C5"}[args.config], wl.height, wl.width,
                           " (one %d-row slab per GPU)" % wl.A if args.scaling == "weak" else " row-split over the GPUs",
                           wl.L, wl.mesh.num_triangles, "+".join(stages)),
            "atlas": [wl.height, wl.width], "layers": wl.L, "triangles": wl.mesh.num_triangles,
            "window": [wl.cam.height, wl.cam.width], "stages": list(stages), "batch_strokes": wl.K,
            "l2": "no explicit flush: every streamed input plane (>= 268 MB) is larger than the 126 MB L2, and the "
                  "streaming stages (chain, mask_op, threshold, area: >= 0.8 GB each, 10 GB together) run between the "
                  "footprint-culled brush stages of consecutive iterations, which therefore start from a cold L2",
            "parallelism": "row-sharded x%d (%s scaling)" % (args.gpus, args.scaling)}


# ------------------------------------------------------------------------------------------------
# GPU arm

class GpuArm:
    """All resident state of one rank and the stage calls through the public API."""

    def __init__(self, args, wl, rank, world_size, dev):
        import torch
        import paper_2501_14807_b200 as ml
        from paper_2501_14807_b200 import _native as nat, sharding
        self.torch, self.ml, self.nat, self.sharding = torch, ml, nat, sharding
        self.args, self.wl, self.rank, self.ws, self.dev = args, wl, rank, world_size, dev
        L, W = wl.L, wl.width
        self.row0, self.rows = sharding.shard_rows(wl.height, world_size, rank)
        rows = self.rows
        self.n = rows * W
        t0 = time.time()
        self.surf = ml.build_surface_map(wl.mesh, W, wl.height, row0=self.row0, rows=rows, device=dev)
        self.need_stroke = any(s in args.stages.split(",") for s in ("tea", "tpa"))
        if self.need_stroke:
            self.depth = ml.render_depth(wl.mesh, wl.cam, device=dev)
            self.ctx = ml.StrokeContext(wl.mesh, wl.cam, self.depth, self.surf, device=dev)
        pool = ml.TexturePool(budget_texels=(2 * L + 8) * self.n + 1, device=dev)
        self.layers = [ml.create_layer("L%d" % i, "uint8", W, rows, pool=pool) for i in range(L)]
        self.out_layer = ml.create_layer("out", "uint8", W, rows, pool=pool)
        self.edited = [torch.zeros((rows, W), dtype=torch.uint8, device=dev) for _ in range(L)]
        self.tmp_mask = torch.zeros((rows, W), dtype=torch.uint8, device=dev)
        # TPA outline, built once per mesh; neighbour slabs supply the 1-row halo
        cov_ext, cov_row0 = sharding.exchange_halo(self.surf.coverage.to(torch.uint8), self.row0, wl.height, 1)
        self.outline = nat.outline_mask(cov_ext, 1, in_row0=cov_row0, out_row0=self.row0, out_rows=rows)
        del cov_ext
        self.batch = nat.StrokeBatch([l.data for l in self.layers], [l.mask for l in self.layers], self.edited, dev,
                                     capacity=wl.K)
        self.attr = self.surf.pos[2]
        self.attr_tiles = nat.attr_tiles(self.attr)     # per-tile height ranges for the culled threshold selection
        self.tool_shape_dev = nat._as_dev_bytes(wl.tool_shape, dev)
        # cross-rank area sum: fused into the reduction kernel over peer memory (sharding.PeerAreaReducer: system-scope
        # atomics into every rank's row, no collective call); ML_AREA_REDUCE=gather, or a node without CUDA IPC, uses
        # the one-all-gather form (sharding.AreaReducer)
        self.area_reduce = sharding.AreaReducer(L, dev)
        self.peer_areas, self.area_step = None, 0
        self.area_reduce_kind = "none (1 rank)" if world_size == 1 else "all-gather"
        if world_size > 1 and os.environ.get("ML_AREA_REDUCE", "peer") == "peer":
            # every rank walks the same sequence of collectives whatever fails locally: the constructor votes after
            # mapping the peers (raising on ALL ranks or none), the trial reduction is bounded by its 10 s wait
            passed = False
            try:
                self.peer_areas = sharding.PeerAreaReducer(L, dev)
            except Exception as exc:                         # e.g. IPC not permitted in this container
                sys.stderr.write("peer area reduction unavailable (%s); using the all-gather form\n" % exc)
            if self.peer_areas is not None:
                try:
                    passed = self.peer_areas.self_test()
                except Exception as exc:
                    sys.stderr.write("peer area self-test failed (%s); using the all-gather form\n" % exc)
                if sharding.agree(passed, dev):               # all ranks or none
                    self.area_reduce_kind = "fused: system-scope atomics into every rank's row over peer memory"
                else:
                    self.peer_areas.close()
                    self.peer_areas = None
        self.T = wl.mesh.num_triangles
        self.seed()
        torch.cuda.synchronize()
        self.setup_s = time.time() - t0
        # result slots of one step (8-byte elements): tea (edited, fragments) | tpa | sphere | threshold | batch [L] |
        # area sums [L] (float64 bit patterns) | area counts [L]
        self.slot = {"tea": (0, 2), "tpa": (2, 3), "sphere": (3, 4), "threshold": (4, 5), "batch": (5, 5 + L),
                     "area": (5 + L, 5 + 3 * L)}
        self.nslots = 5 + 3 * L

    def seed(self):
        """(Re)create the pre-painted state: empty planes, then 4 seeded sphere strokes per layer."""
        ml, wl = self.ml, self.wl
        for l in self.layers + [self.out_layer]:
            l.data.zero_()
            l.mask.zero_()
        for e in self.edited:
            e.zero_()
        self.tmp_mask.zero_()
        if self.need_stroke:
            self.ctx.edited.zero_()
            self.ctx.edited_fully_dirty = True          # the next culled stroke resets its tile buffers
        for k in range(len(wl.seed_strokes)):
            ml.select_sphere(self.surf, self.layers[k % wl.L], wl.seed_strokes[k, :3], wl.seed_strokes[k, 3],
                             wl.seed_labels[k], edited=self.edited[k % wl.L])

    def culled(self, cull):
        return cull and self.surf.tiles is not None

    def launches(self, cull):
        c = self.culled(cull)
        return {"tea": 3, "tpa": 1, "sphere": 2 if c else 1, "batch": 2 if c else 1, "chain": 1, "mask_op": 1,
                "threshold": 2 if (c and self.attr_tiles is not None) else 1, "area": -(-self.wl.L // 8)}

    def make_tool(self, inp):
        return self.ml.EditingTool(px=float(inp["tool_xy"][0]), py=float(inp["tool_xy"][1]), shape=self.tool_shape_dev, value=7)

    def stage(self, st, inp, tool, row, cull):
        """Queue one stage through the public API.  Its counters accumulate into the (zeroed) slots of `row`, an
        int64 device vector of `nslots` elements; nothing here synchronises or allocates."""
        ml, nat, wl, L = self.ml, self.nat, self.wl, self.wl.L
        layers, edited = self.layers, self.edited
        a, b = self.slot.get(st, (0, 0))
        if st == "tea":
            ml.apply_stroke(self.ctx, tool, layers[0], eps=wl.eps, cull=cull, counts=row[a:b])
        elif st == "tpa":
            # padding of the stroke just applied (the paper times TEA + TPA per edit); with
            # several ranks the 1-row halo of the edited plane travels point-to-point first
            tiles = self.ctx.stroke_tiles if cull else None
            if self.ws > 1:
                ml.editing.pad_slab(self.outline, self.ctx.edited, 1, layers[0].data, layers[0].mask, tool.value, row[a:b],
                                    row0=self.row0, height=wl.height, tiles=tiles, ext=self.ctx.edited_ext)
            else:
                nat.apply_padding(self.outline, self.ctx.edited, 1, layers[0].data, layers[0].mask, tool.value,
                                  counts=row[a:b], tiles=tiles)
        elif st == "sphere":
            s = inp["sphere"]
            ml.select_sphere(self.surf, layers[1 % L], s[:3], s[3], inp["sphere_value"], edited=edited[1 % L], cull=cull,
                             counts=row[a:b])
        elif st == "batch":
            self.batch.counts = row[a:b]
            ml.select_sphere_batch(self.surf, self.batch, cull=cull)
        elif st == "chain":
            ml.layer_chain(layers[:wl.chain_n], wl.chain_ops, self.out_layer, lazy=cull)
        elif st == "mask_op":
            nat.layer_op("union", None, layers[0].mask, None, layers[1 % L].mask, None, self.tmp_mask)
        elif st == "threshold":
            ml.select_threshold(self.attr, None, wl.thr[0], wl.thr[1], layers[2 % L], inp["thr_value"], edited=edited[2 % L],
                                tiles=self.attr_tiles if cull else None, counts=row[a:b])
        elif st == "area":
            if self.peer_areas is not None:
                self.peer_areas.reduce(self.area_step, self.surf.area, [l.mask for l in layers], row[a:b])
                self.area_step += 1
            else:
                nat.layer_area(self.surf.area, [l.mask for l in layers], sums=row[a:a + L].view(self.torch.float64),
                               counts=row[a + L:b])
                self.area_reduce(row[a:b])

    def hits_of(self, st, row_host):
        a, b = self.slot[st]
        return float(row_host[a]) if st != "batch" else float(row_host[a:b].sum())


def run_ours(args):
    import torch
    import paper_2501_14807_b200 as ml
    from paper_2501_14807_b200 import _native as nat

    rank = int(os.environ.get("RANK", "0"))
    world_size = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    nat.require_cuda()
    # ML_BENCH_BACKEND=gloo is a TEST hook: it lets several ranks share one GPU (NCCL refuses that) so
    # the multi-rank code path can be exercised on a single-GPU box; the measured runs use NCCL
    backend = os.environ.get("ML_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world_size > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    stages = [s for s in args.stages.split(",") if s]
    wl = Workload(args, world_size)
    arm = GpuArm(args, wl, rank, world_size, dev)
    L, n, T = wl.L, arm.n, arm.T
    primary_cull = not args.no_cull

    def barrier():
        if world_size > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world_size == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    total_steps = args.warmup + args.steps
    inputs = [wl.step_inputs(i) for i in range(total_steps)]
    # ONE counter block per loop, zeroed once: row k holds every stage's results of step k
    slots = torch.zeros((total_steps, arm.nslots), dtype=torch.int64, device=dev)

    # Resident loops: EVERY step has its own strokes (tool position, sphere stroke, batch table); the batch tables of all
    # steps are uploaded once, before the timed regions, and a step binds its table by pointer.  (Re-applying one table
    # every step would let the batch kernel skip its stores from the second step on -- texels already hold the value.)
    tables = None
    if "batch" in stages:
        nb = wl.K * nat.StrokeBatch.RECORD_BYTES
        host_tables = np.zeros((total_steps, nb), np.uint8)
        for i in range(total_steps):
            arm.batch.pack_host(inputs[i]["batch"], inputs[i]["batch_layers"], inputs[i]["batch_values"], host_tables[i])
        tables = torch.from_numpy(host_tables).to(dev)
        if world_size > 1:
            import torch.distributed as dist
            dist.broadcast(tables, src=0)

    # clock sampler: started before the warm-up so that nvidia-smi is already delivering samples when the
    # timed region begins (its start-up alone can outlast a short timed region)
    stop, samples, windows = threading.Event(), [], []
    th = threading.Thread(target=sample_clocks, args=(stop, samples), daemon=True)
    th.start()
    t_wait = time.time()
    while not samples and time.time() - t_wait < 5.0 and th.is_alive():
        time.sleep(0.02)

    def resident_loop(cull):
        """W warm-up + K timed steps, everything resident, no read-back.  Returns (total ms, per-stage ms, host rows)."""
        slots.zero_()
        for i in range(args.warmup):
            tool = arm.make_tool(inputs[i])
            if "batch" in stages:
                arm.batch.bind(tables[i], wl.K)
            for st in stages:
                arm.stage(st, inputs[i], tool, slots[i], cull)
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(stages) + 1)] for _ in range(args.steps)]
        barrier()
        t_begin = time.time()
        for k in range(args.steps):
            inp = inputs[args.warmup + k]
            tool = arm.make_tool(inp)
            row = slots[args.warmup + k]
            if "batch" in stages:
                arm.batch.bind(tables[args.warmup + k], wl.K)      # this step's strokes (resident since before the loop)
            ev[k][0].record()
            for j, st in enumerate(stages):
                arm.stage(st, inp, tool, row, cull)
                ev[k][j + 1].record()
        barrier()
        windows.append((t_begin, time.time()))
        total_ms = max_over_ranks(ev[0][0].elapsed_time(ev[-1][-1]))
        stage_ms = {st: sum(ev[k][j].elapsed_time(ev[k][j + 1]) for k in range(args.steps)) / args.steps
                    for j, st in enumerate(stages)}
        return total_ms, stage_ms, slots[args.warmup:].cpu().numpy()

    if args.profile_loop:
        t_ms, s_ms, _ = resident_loop(args.profile_loop == "default")
        stop.set()
        th.join()
        if rank == 0:
            print(json.dumps({"profile_loop": args.profile_loop, "steps": args.steps, "warmup": args.warmup,
                              "ms_per_step": t_ms / args.steps, "stage_ms": {k: round(v, 4) for k, v in s_ms.items()},
                              "launches_per_step": sum(arm.launches(args.profile_loop == "default")[s] for s in stages)}))
        return
    # ---- value: the default path;  value_streamed: every stage streams the whole atlas
    total_ms, stage_ms, _ = resident_loop(primary_cull)
    if primary_cull:
        total_ms_s, stage_ms_s, _ = resident_loop(False)
    else:
        total_ms_s, stage_ms_s = total_ms, stage_ms

    # ---- e2e loop: the default path, but every step (1) takes its stroke records from HOST memory (pinned
    # staging -> device) and (2) reads the step's result row (edit counts, padded count, per-layer areas and
    # texel counts) back to the host: one non-blocking copy into pinned memory queued behind the step's last
    # stage, consumed by the host after the FIRST stage of the next step has been queued (the GPU never waits
    # for the host between steps; the last step's row is consumed before the closing event).
    pinned_in = torch.empty(16, dtype=torch.float64).pin_memory()
    rec_dev = torch.empty(16, dtype=torch.float64, device=dev)
    out_pinned = [torch.empty(arm.nslots, dtype=torch.int64).pin_memory() for _ in range(2)]
    pending = []

    def consume():
        got = 0
        while pending:
            e, nbytes = pending.pop(0)
            e.synchronize()             # the host now holds that step's results in pinned memory
            got += nbytes
        return got

    # Host <-> device copies of the e2e loop run on a SIDE stream: a copy queued in the compute stream costs two
    # engine hand-overs (kernel -> copy engine -> kernel, ~35 us each way around the 320-byte stroke table: measured
    # 0.076 ms per step), so the step's inputs go up beside the first stages and the compute stream only waits for
    # their event before the kernel that reads them; the result row goes down beside the next step's first stage.
    main_stream = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    step_done = [torch.cuda.Event(), torch.cuda.Event()]

    def e2e_step(idx, slot):
        inp = inputs[idx]
        rec = np.concatenate([inp["tool_xy"], inp["sphere"]])
        pinned_in[:rec.size].copy_(torch.from_numpy(rec))
        with torch.cuda.stream(side):
            rec_dev[:rec.size].copy_(pinned_in[:rec.size], non_blocking=True)   # this step's scalar stroke record
            if "batch" in stages and rank == 0:
                # this step's stroke table: pinned host memory -> the device copy no queued kernel is reading
                arm.batch.upload(inp["batch"], inp["batch_layers"], inp["batch_values"], fill=world_size > 1)
        tool = arm.make_tool(inp)
        row = slots[idx]
        got = 0
        for j, st in enumerate(stages):
            if st == "batch":
                if rank == 0:
                    main_stream.wait_event(arm.batch.ready)
                arm.sharding.broadcast_batch(arm.batch)          # one device broadcast to the other ranks (no-op at N = 1)
            arm.stage(st, inp, tool, row, primary_cull)
            if j == 0:
                got += consume()        # results of the previous step
        step_done[slot].record(main_stream)
        with torch.cuda.stream(side):
            side.wait_event(step_done[slot])
            out_pinned[slot].copy_(row, non_blocking=True)
            e = torch.cuda.Event()
            e.record(side)
        pending.append((e, 8 * arm.nslots))
        return got

    slots.zero_()
    for i in range(args.warmup):
        e2e_step(i, i & 1)
    consume()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_begin = time.time()
    e0.record()
    d2h = 0
    for k in range(args.steps):
        d2h += e2e_step(args.warmup + k, k & 1)
    d2h += consume()
    e1.record()
    barrier()
    windows.append((t_begin, time.time()))
    e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    h2d = 8 * 6 + 64 + (wl.K * nat.StrokeBatch.RECORD_BYTES if "batch" in stages else 0)   # stroke records + 4x4 matrix

    # ---- e2e_host_planes: the reference's call shape (KN:135-136) per step -- numpy planes in pageable host
    # memory, the drop-in twin uploads the triangle arrays, runs the direct kernel and writes the stroke's
    # texels back into the caller's planes, all inside the timed region
    host_planes = None
    if rank == 0 and world_size == 1 and not args.no_cpu and "tea" in stages and args.host_plane_reps > 0:
        W, rows = wl.width, arm.rows
        tri_xy = np.ascontiguousarray(wl.mesh.tri_uv_texels(W, wl.height))
        clip = np.ascontiguousarray(wl.cam.clip_coords(wl.mesh.vertices)[wl.mesh.triangles])
        depth_np = arm.depth.plane.cpu().numpy()
        shape_np = np.ascontiguousarray(wl.tool_shape).astype(np.uint8)
        planes = [np.zeros((rows, W), np.uint8) for _ in range(3)]
        t_calls, last = [], None
        for r in range(args.host_plane_reps + 1):
            inp = inputs[args.warmup + (r % args.steps)]
            tool = arm.make_tool(inp)
            sfx, sfy, bx, by = ml.compute_tool_projection(wl.cam, tool).kernel_factors
            planes[2][:] = 0                                            # EditedAreaMask reset, host side
            t0 = time.perf_counter()
            last = nat.raster_tea(tri_xy, clip, float(wl.cam.width), float(wl.cam.height), depth_np, wl.eps, sfx, sfy,
                                  bx, by, shape_np, planes[0], planes[1], planes[2], 7)
            t_calls.append((time.perf_counter() - t0) * 1e3)
        windows.append((time.time() - sum(t_calls) * 1e-3, time.time()))
        # same stroke through the resident engine: counts must agree
        chk = torch.zeros(2, dtype=torch.int64, device=dev)
        arm.ctx.edited.zero_()
        arm.ctx.edited_fully_dirty = True
        lay = arm.out_layer
        lay.data.zero_(); lay.mask.zero_()
        ml.apply_stroke(arm.ctx, arm.make_tool(inputs[args.warmup + ((args.host_plane_reps) % args.steps)]), lay,
                        eps=wl.eps, counts=chk)
        same = (int(chk[0].item()) == int(last[0]) and
                np.array_equal(lay.mask.cpu().numpy().view(np.uint8) != 0, planes[2] != 0))
        ms = float(np.median(t_calls[1:]))
        naive = tri_xy.nbytes + clip.nbytes + depth_np.nbytes + shape_np.nbytes + 6 * planes[0].nbytes
        host_planes = {"op": "raster_tea (KN:135-136) with numpy planes in pageable host memory, per call: pipelined upload "
                             "of the triangle arrays + direct per-triangle kernel + sparse write-back of the stroke's texels",
                       "ms_per_call": round(ms, 3), "first_call_ms": round(t_calls[0], 2), "calls": args.host_plane_reps,
                       "value": n / (ms * 1e-3) / 1e9, "unit": "Gtexel/s",
                       "h2d_bytes_per_call": int(tri_xy.nbytes + clip.nbytes + depth_np.nbytes + shape_np.nbytes),
                       "d2h_bytes_per_call": "O(hit texels / 8): the written SET as a bitmap or word list",
                       "plane_round_trip_bytes_avoided": int(naive), "edited": int(last[0]), "fragments": int(last[1]),
                       "equal_to_resident_stroke": bool(same)}
        # the other two reference call shapes, same conditions: coverage_fill (KN:84) into a zeroed 16384^2 host
        # plane and raster_depth (KN:103) into a host depth plane pre-filled with 1.0
        from paper_2501_14807_b200.mesh_core import window_triangles
        cov = planes[0]
        t_cov = []
        for r in range(3):
            cov[:] = 0
            t0 = time.perf_counter()
            written = nat.coverage_fill(tri_xy, W, rows, cov)
            t_cov.append((time.perf_counter() - t0) * 1e3)
        wxy, wzn = window_triangles(wl.mesh, wl.cam)
        t_dep = []
        for r in range(3):
            dplane = np.ones((wl.cam.height, wl.cam.width), np.float32)
            t0 = time.perf_counter()
            nat.raster_depth(wxy, wzn, dplane)
            t_dep.append((time.perf_counter() - t0) * 1e3)
        host_planes["coverage_fill_ms_per_call"] = round(float(np.median(t_cov[1:])), 3)
        host_planes["coverage_fill_equals_surface_map"] = bool(int(written) == arm.surf.covered)
        host_planes["raster_depth_ms_per_call"] = round(float(np.median(t_dep[1:])), 3)
        host_planes["raster_depth_equals_resident"] = bool(np.array_equal(dplane.view(np.uint32), depth_np.view(np.uint32)))
        del planes, tri_xy, clip
    stop.set()
    th.join()

    # ---- hit census (untimed): mean number of texels each brush stage writes per step, for the
    # hit-write term of the algorithmic bytes.  Edited planes are cleared first so that the
    # kernels' "newly edited" counters equal the hit counts.
    hits = {s: 0.0 for s in stages}
    ncen = min(args.steps, 10)
    slots.zero_()
    for k in range(ncen):
        inp = inputs[args.warmup + k]
        tool = arm.make_tool(inp)
        for e in arm.edited:
            e.zero_()
        if "batch" in stages:
            arm.batch.bind(tables[args.warmup + k], wl.K)
        for st in stages:
            arm.stage(st, inp, tool, slots[k], primary_cull)
    census = slots[:ncen].cpu().numpy()
    for st in stages:
        if st in BRUSH:
            hits[st] = float(np.mean([arm.hits_of(st, census[k]) for k in range(ncen)]))

    # ---- whole-atlas streaming form of every stage, alone inside a CUDA graph (no host launch latency)
    stream_kernels = {}
    peak, peak_src = measured_peak()
    if rank == 0 and world_size == 1:
        inp = inputs[args.warmup]
        tool = arm.make_tool(inp)
        scratch_row = torch.zeros(arm.nslots, dtype=torch.int64, device=dev)
        if "tpa" in stages:
            arm.stage("tea", inp, tool, scratch_row, False)              # marks for the padding pass
        for st in stages:
            ms, graphed = time_graph(lambda: arm.stage(st, inp, tool, scratch_row, False), inner=10, reps=5)
            b = wl.algorithmic_bytes(n, st, T, hits[st])
            stream_kernels[st] = {"ms": round(ms, 4), "gb_s": round(b / ms / 1e6, 1), "frac_of_peak": round(b / ms / 1e6 / peak, 4),
                                  "timed": "cuda graph of 10 calls" if graphed else "eager back-to-back calls"}

        if "tea" in stages:
            # the id stream of the whole-atlas TEA stage alone: a tool far outside the window flags no triangle, so the
            # stage is classification + id stream with the edited reset + an empty evaluation launch (5 B/texel); the
            # difference to "tea" above is the float64 evaluation of the 70 px tool's footprint
            off_tool = ml.EditingTool(px=-1.0e6, py=-1.0e6, shape=arm.tool_shape_dev, value=7)
            ms, graphed = time_graph(lambda: arm.stage("tea", inp, off_tool, scratch_row, False), inner=10, reps=5)
            b = wl.algorithmic_bytes(n, "tea", T, 0)
            stream_kernels["tea_id_stream_only"] = {"ms": round(ms, 4), "gb_s": round(b / ms / 1e6, 1),
                                                    "frac_of_peak": round(b / ms / 1e6 / peak, 4),
                                                    "timed": "cuda graph of 10 calls" if graphed else "eager back-to-back calls",
                                                    "note": "tool outside the window: no triangle flagged, nothing to evaluate"}

    # ---- parity (untimed) + cpu_baseline
    parity, cpu = None, None
    if rank == 0 and world_size == 1 and not args.no_cpu:
        cpu_arm = CpuArm(wl, args.cpu_rows)
        parity = parity_check(arm, cpu_arm, wl, stages, args.parity_steps)
        cpu_arm.step(0, stages)
        reps, el, per = 0, 0.0, {s: 0.0 for s in stages}
        while reps < 3 or (el < 10.0 and reps < 20):
            t, _ = cpu_arm.step(1 + reps, stages)
            for s in stages:
                per[s] += t[s]
            el += sum(t.values())
            reps += 1
        cpu = {"value": len(stages) * cpu_arm.n * reps / el / 1e9, "unit": "Gtexel/s", "cores": cpu_arm.threads, "kind": "port",
               "sample": "%d of %d rows of the slab (%.1f Mtexel) x %d reps; %s" % (cpu_arm.rows, wl.A, cpu_arm.n / 1e6, reps,
                                                                                      CpuArm.DESCRIPTION),
               "stage_ms": {s: round(per[s] / reps * 1e3, 3) for s in stages}, "threads": cpu_arm.threads}

    # ---- report
    traffic = {}
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f)

    def stage_table(ms_of, cull):
        """Per stage: time, algorithmic GB/s and fraction; DRAM bytes per step (ncu capture of the stage's kernels,
        per launch x launches) and the fraction of the peak they amount to in the measured time."""
        out = {}
        launches = arm.launches(cull)
        for st in stages:
            b = wl.algorithmic_bytes(n, st, T, hits[st])
            ms = ms_of[st]
            row = {"ms": round(ms, 4), "gtexel_s": round(n / (ms * 1e-3) / 1e9, 2), "alg_bytes": b,
                   "gb_s": round(b / ms / 1e6, 1), "frac_of_peak": round(b / ms / 1e6 / peak, 4),
                   "hits_per_step": int(hits[st]), "launches": launches[st]}
            key = st if arm.culled(cull) or st in ("mask_op", "area") else st + "_stream"
            if st == "chain":
                key = "chain" if cull else "chain_stream"
            tb = traffic.get(key)
            if tb is not None:
                # traffic.json: DRAM bytes of one launch of each of the stage's kernels in the default workload
                # (16384^2 texels, 8 layers); other atlas sizes scale with the texel count, more layers with the
                # number of 8-layer area launches
                per_step = tb * (launches[st] if st == "area" else 1) * n / float(traffic.get("_texels", 16384 * 16384))
                row["dram_bytes"] = per_step
                row["dram_frac_of_peak"] = round(per_step / ms / 1e6 / peak, 4)
            if st in BRUSH:
                row["footprint_culled"] = bool(arm.culled(cull))
            if st == "chain":
                row["lazy_data_reads"] = bool(cull)
            out[st] = row
        return out

    texel_passes = len(stages) * n * world_size
    value = texel_passes * args.steps / (total_ms * 1e-3) / 1e9
    value_s = texel_passes * args.steps / (total_ms_s * 1e-3) / 1e9
    e2e_value = texel_passes * args.steps / (e2e_ms * 1e-3) / 1e9
    tab, tab_s = stage_table(stage_ms, primary_cull), stage_table(stage_ms_s, False)

    def roof(tab_x, ms_x, note):
        dom = max(stages, key=lambda s: ms_x[s])
        r = tab_x[dom]
        out = {"bound": "hbm", "kernel": dom, "achieved": r["alg_bytes"] / ms_x[dom] / 1e6, "peak": peak, "unit": "GB/s",
               "frac": r["alg_bytes"] / ms_x[dom] / 1e6 / peak, "traffic": r.get("dram_bytes"),
               "dram_achieved": None if "dram_bytes" not in r else r["dram_bytes"] / ms_x[dom] / 1e6,
               "dram_frac": r.get("dram_frac_of_peak"), "stage_ms": round(ms_x[dom], 4),
               "frac_of_8TBs_spec": r["alg_bytes"] / ms_x[dom] / 1e6 / 8000.0, "basis": note}
        return out

    if rank == 0:
        cfg = workload_config(args, wl, stages)
        cfg["stage_results"] = tab
        cfg["stage_results_streamed"] = tab_s
        cfg["stream_kernels"] = stream_kernels
        cfg["setup_s"] = round(arm.setup_s, 2)
        cfg["surface_map"] = {"covered": arm.surf.covered, "overlap": arm.surf.overlap}
        cfg["footprint_culling"] = bool(arm.culled(primary_cull))
        cfg["area_reduce"] = arm.area_reduce_kind
        cfg["value_basis"] = ("value counts NOMINAL texel passes (stages x slab texels) of the default path, whose brush / selection stages "
                              "and chain skip most of their bytes by design; value_streamed is the same step with every stage reading "
                              "its whole atlas (byte-honest); both from CUDA events over the same %d steps" % args.steps)
        roofline = roof(tab, stage_ms, "slowest stage of the default step: SURVEY 8(d) algorithmic bytes / CUDA-event time "
                                       "(frac); dram_frac = ncu-measured DRAM bytes of the stage's kernels / the same time. "
                                       "A stage that skips bytes by design (culled brushes, lazy chain, sparse-mask area) shows "
                                       "frac > dram_frac; roofline.streamed is the byte-honest twin")
        roofline["peak_source"] = peak_src
        roofline["streamed"] = roof(tab_s, stage_ms_s, "slowest stage of the streamed step (every stage reads its whole atlas)")
        out = {
            "metric": "brush-apply + layer-op texel passes per second at 16384^2 atlas",
            "value": value, "unit": "Gtexel/s", "n_gpus": world_size, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64 decisions on u8/u32/f32 planes", "data": "synthetic", "config": cfg,
            "value_streamed": value_s, "ms_per_step_streamed": total_ms_s / args.steps,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "Gtexel/s", "ms_per_step": e2e_ms / args.steps,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h // max(1, args.steps)},
            "e2e_host_planes": host_planes,
            "parity": parity,
            "gpu_launches": sum(arm.launches(primary_cull)[s] for s in stages) * args.steps,
            "clocks": clocks_summary(samples, windows),
        }
        print(json.dumps(out))
    if arm.peer_areas is not None:
        arm.peer_areas.check()
    if world_size > 1:
        import torch.distributed as dist
        dist.barrier()
        if arm.peer_areas is not None:
            arm.peer_areas.close()
        dist.destroy_process_group()
    if parity is not None and not parity["ok"]:
        sys.exit(3)


def parity_check(arm, cpu_arm, wl, stages, steps):
    """GPU arm vs CPU arm on the same seeded inputs.  Both start from the pre-painted state and run `steps`
    steps; the GPU does it twice (default path, then every stage streaming the whole atlas).  Compared on the
    CPU arm's rows minus one border row each side (the CPU slab has no halo for the 1-texel TPA stencil):
    data / mask / edited planes of all layers, the stroke's EditedAreaMask, the chain result, the mask_op result
    (bit for bit) and the per-layer areas and texel counts of those rows (1e-10 relative; north star: 1e-6)."""
    torch, nat = arm.torch, arm.nat
    r0, r1 = cpu_arm.row0 + 1, cpu_arm.row0 + cpu_arm.rows - 1
    lo, hi = 1, cpu_arm.rows - 1
    report = {"checked": True, "ok": True, "rows": [r0, r1], "steps": steps, "stages": list(stages), "paths": {},
              "against": CpuArm.DESCRIPTION}
    for i in range(steps):
        cpu_arm.step(i, stages)
    cpu_planes = {}
    for k in range(wl.L):
        cpu_planes["data%d" % k], cpu_planes["mask%d" % k], cpu_planes["edited%d" % k] = cpu_arm.data[k], cpu_arm.mask[k], cpu_arm.edited[k]
    if "tea" in stages:
        cpu_planes["tea_edited"] = cpu_arm.tea_edited
    if "chain" in stages:
        cpu_planes["chain_data"], cpu_planes["chain_mask"] = cpu_arm.out_d, cpu_arm.out_m
    if "mask_op" in stages:
        cpu_planes["mask_op"] = cpu_arm.tmp_m
    cpu_area = cpu_arm.kn.layers_area(np.ascontiguousarray(cpu_arm.surf["area"][lo:hi]),
                                      [np.ascontiguousarray(m[lo:hi]) for m in cpu_arm.mask], threads=cpu_arm.threads)
    snap = None
    for path, cull in (("default", True), ("streamed", False)):
        arm.seed()
        rows_t = torch.zeros((steps, arm.nslots), dtype=torch.int64, device=arm.dev)
        for i in range(steps):
            inp = wl.step_inputs(i)
            tool = arm.make_tool(inp)
            if "batch" in stages:
                arm.batch.upload(inp["batch"], inp["batch_layers"], inp["batch_values"])
            for st in stages:
                arm.stage(st, inp, tool, rows_t[i], cull)
        gpu = {}
        for k in range(wl.L):
            gpu["data%d" % k], gpu["mask%d" % k], gpu["edited%d" % k] = arm.layers[k].data, arm.layers[k].mask, arm.edited[k]
        if "tea" in stages:
            gpu["tea_edited"] = arm.ctx.edited
        if "chain" in stages:
            gpu["chain_data"], gpu["chain_mask"] = arm.out_layer.data, arm.out_layer.mask
        if "mask_op" in stages:
            gpu["mask_op"] = arm.tmp_mask
        bad = []
        for name, t in gpu.items():
            g = t[r0 - arm.row0:r1 - arm.row0].cpu().numpy().view(np.uint8)
            if not np.array_equal(g, np.ascontiguousarray(cpu_planes[name][lo:hi]).view(np.uint8)):
                bad.append(name)
        sums = torch.zeros(wl.L, dtype=torch.float64, device=arm.dev)
        cnts = torch.zeros(wl.L, dtype=torch.int64, device=arm.dev)
        nat.layer_area(arm.surf.area[r0 - arm.row0:r1 - arm.row0], [l.mask[r0 - arm.row0:r1 - arm.row0] for l in arm.layers],
                       sums=sums, counts=cnts)
        gs, gc = sums.cpu().numpy(), cnts.cpu().numpy()
        rel = float(np.max(np.abs(gs - cpu_area[0]) / np.maximum(np.abs(cpu_area[0]), 1e-300)))
        if not np.array_equal(gc, cpu_area[1]) or not rel <= 1e-10:
            bad.append("areas")
        # whole-plane agreement of the two GPU paths (all rows, on the device)
        if snap is None:
            snap = {k: v.clone() for k, v in gpu.items()}
            counts_default = rows_t.cpu().numpy()
        else:
            for k, v in gpu.items():
                if not torch.equal(v, snap[k]):
                    bad.append("streamed!=default:" + k)
            cs = rows_t.cpu().numpy()
            a, b = arm.slot["area"]
            if not np.array_equal(np.delete(cs, np.s_[a:a + wl.L], axis=1), np.delete(counts_default, np.s_[a:a + wl.L], axis=1)):
                bad.append("streamed!=default:counters")
        report["paths"][path] = {"planes_compared": len(gpu), "texels_per_plane": int((r1 - r0) * wl.width),
                                 "area_max_rel_err": rel, "mismatches": bad}
        if bad:
            report["ok"] = False
    del snap
    arm.seed()
    return report


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
