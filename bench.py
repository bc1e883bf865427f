#!/usr/bin/env python
"""bench.py -- brush-apply + layer-op throughput at a 16384^2 atlas (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One STEP = one pass of every hot-path stage over this rank's 16384 x 16384 atlas slab
(268.4 Mtexel), the C3+C4 workload of BASELINE.json at 8 layers (``--layers 64`` gives C4); the
stages run in the order of ``STAGES`` below (streaming stages first), listed here by kind:

    tea        the paper's projective brush (TEA, KN:135-203) over the cached triangle-id map
    tpa        the paper's padding pass (TPA): outline texels next to the stroke
    sphere     one sphere-brush stroke over the float32x3 position map
    batch      L sphere strokes (one per layer) batched in ONE pass over the position map
               (the brush / selection stages tea, tpa, sphere, batch and threshold run the
               footprint-culled kernels: a stroke reads only the tiles it can reach, the threshold
               only tiles whose height range meets the window, the chain reads a data vector only
               where the masks let it reach the result; ``--no-cull`` streams the whole atlas, and
               the whole-atlas streaming kernels are ALSO timed on their own and reported under
               ``config.stream_kernels`` -- they are the brush kernels' HBM-roofline evidence)
    chain      fused layer-algebra chain ((L0 u L1) n L2) \\ L3 ... over 8 uint8 layers (C3)
    mask_op    binary union of two bare uint8 mask planes (the 3 B/texel streaming kernel)
    threshold  attribute-threshold selection on the float32 attribute plane pos.z (C3)
    area       per-layer area of all L layers in one fused pass (+ NCCL all-reduce when N > 1)

metric = texel passes per second: (stages x slab texels x ranks) / step time, in Gtexel/s.
Inputs are far larger than the 126 MB L2 (every plane is >= 268 MB), so no explicit L2 flush is
needed between iterations.  ``value`` is timed with CUDA events with everything resident in HBM;
``e2e`` runs the same step through the public API from HOST stroke records (pinned memory ->
device every step) and reads every stage's result (edit counts, areas) back to the host every step
(one non-blocking copy into pinned memory queued behind the step's last stage, consumed by the host
once the next step's first stage has been queued -- the GPU never waits for the host between steps).
``config.host_plane_call`` additionally times ONE drop-in call of the KN twin ``raster_tea`` with numpy
planes in host memory (upload + kernel + download inside the call, the way the reference's numpy
backend is called): the PCIe cost the resident design exists to avoid, reported beside ``e2e``.

Multi-GPU (torchrun, one rank per GPU): weak scaling -- the atlas grows to 16384 x (16384*N) and
each rank owns one 16384-row slab; the only collectives are the stroke broadcast and the area
all-reduce (scalars).

``--impl reference`` times the reference-side CPU implementation (oracle/kn_port.c, the C
restatement of the reference's numpy kernels, row-parallel over all host threads) on a bounded
row sample of the same workload.
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--atlas", type=int, default=16384, help="atlas width and per-rank slab height")
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--quads", type=int, default=707, help="heightfield quads per side (707 -> 999,698 tris)")
    ap.add_argument("--window", type=int, default=1024)
    ap.add_argument("--cpu-rows", type=int, default=1024, help="rows of the slab the CPU baseline processes")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-cull", action="store_true",
                    help="every stage streams the whole atlas: brush / selection stages ignore their footprint tiles, the "
                         "chain reads every data vector")
    ap.add_argument("--stages", default=",".join(STAGES))
    return ap.parse_args()


# ------------------------------------------------------------------------------------------------
# workload definition shared by both arms

class Workload:
    def __init__(self, args, world_size):
        from paper_2501_14807_b200 import synth
        self.A = args.atlas
        self.width, self.height = args.atlas, args.atlas * world_size
        self.L = args.layers
        self.mesh = synth.heightfield_mesh(args.quads, margin=0.01)   # 1% uv border: a real island outline for TPA
        self.cam = synth.default_camera(args.window, args.window, eye=(0.5, 0.5, 1.6), target=(0.5, 0.5, 0.0),
                                        fovy=40.0, near=0.2, far=5.0)
        self.tool_shape = synth.circle_shape(70)                     # the paper's mid radius (70 px)
        self.eps = 1e-4
        rng = np.random.default_rng(synth.SEED + 7)
        self.rng = rng
        nchain = min(8, self.L)
        self.chain_n = nchain
        self.chain_ops = CHAIN_OPS[:nchain - 1]
        z = self.mesh.vertices[:, 2]
        self.thr = (float(np.percentile(z, 40.0)), float(np.percentile(z, 60.0)))   # C3 window
        # per-step host inputs (seeded): tool position, sphere stroke, batch strokes
        self.seed_strokes, self.seed_labels = synth.sphere_strokes(self.mesh, 4 * self.L, seed=synth.SEED + 3,
                                                                   rmin_frac=0.02, rmax_frac=0.08)

    def step_inputs(self, i):
        from paper_2501_14807_b200 import synth
        rng = np.random.default_rng(synth.SEED + 100 + i)
        w = self.cam.width
        tool_xy = rng.uniform(0.3 * w, 0.7 * w, size=2)
        strokes, labels = synth.sphere_strokes(self.mesh, self.L + 1, seed=synth.SEED + 1000 + i,
                                               rmin_frac=0.01, rmax_frac=0.05)
        return dict(tool_xy=tool_xy, sphere=strokes[0], sphere_value=int(labels[0]),
                    batch=strokes[1:], batch_layers=np.arange(self.L, dtype=np.int32), batch_values=labels[1:])

    def algorithmic_bytes(self, n, stage, T, hits=0):
        """Algorithmic HBM bytes of one stage over n texels: the read stream plus,
        for the brushes, `hits` texels x (1 B edited read + 1 B edited + 1 B mask + 1 B uint8 data
        written).  tea additionally resets the 1 B/texel edited plane and reads the
        clip coordinates of every triangle once for the classification pass."""
        L = self.L
        # tea: id stream + edited reset + classification pass; with footprint culling (default) the
        # kernel reads far less than this, so its "frac of peak" can exceed 1 -- the stage is then
        # bound by the float64 evaluation of the footprint, not by HBM
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


# ------------------------------------------------------------------------------------------------
# CPU arm (reference / cpu_baseline): oracle C restatement, all host threads, bounded row sample

class CpuArm:
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
                                   rows=(self.row0, self.row0 + self.rows))
        from paper_2501_14807_b200.mesh_core import window_triangles
        xy, zn = window_triangles(m, wl.cam)
        self.depth = np.ones((wl.cam.height, wl.cam.width), np.float32)
        kn.raster_depth(xy, zn, self.depth, threads=self.threads)
        self.setup_s = time.time() - t0
        n = self.rows * W
        self.n = n
        mk = lambda dt: [np.zeros((self.rows, W), dt) for _ in range(wl.L)]
        self.data, self.mask, self.edited = mk(np.uint8), mk(np.uint8), mk(np.uint8)
        self.out_d, self.out_m = np.zeros((self.rows, W), np.uint8), np.zeros((self.rows, W), np.uint8)
        self.outline = kn.outline((self.surf["tri_id"] >= 0).astype(np.uint8), 1, threads=self.threads)
        self.tmp_d, self.tmp_m = np.zeros((self.rows, W), np.uint8), np.zeros((self.rows, W), np.uint8)
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
                self.edited[0][:] = 0
                res["tea"] = kn.raster_tea_slab(self.tri_xy, self.tri_clip, float(wl.cam.width), float(wl.cam.height),
                                                self.depth, wl.eps, sfx, sfy, bx, by, wl.tool_shape, self.data[0],
                                                self.mask[0], self.edited[0], 7, wl.height, self.row0, th)
            elif st == "tpa":
                res["tpa"] = kn.padding(self.outline, self.edited[0], 1, self.data[0], self.mask[0], 7, threads=th)
            elif st == "sphere":
                s = inp["sphere"]
                res["sphere"] = kn.select_sphere(self.surf["pos"], s[:3], s[3], self.data[1 % wl.L], self.mask[1 % wl.L],
                                                 self.edited[1 % wl.L], inp["sphere_value"], threads=th)
            elif st == "batch":
                res["batch"] = [kn.select_sphere(self.surf["pos"], s[:3], s[3], self.data[L], self.mask[L], self.edited[L],
                                                 v, threads=th)
                                for s, L, v in zip(inp["batch"], inp["batch_layers"], inp["batch_values"])]
            elif st == "chain":
                cd, cm = self.data[0], self.mask[0]
                for j in range(1, wl.chain_n):
                    od, om = (self.out_d, self.out_m) if j % 2 else (self.tmp_d, self.tmp_m)
                    kn.layer_op(wl.chain_ops[j - 1], cd, cm, self.data[j], self.mask[j], od, om, threads=th)
                    cd, cm = od, om
                res["chain"] = (cd, cm)
            elif st == "mask_op":
                kn.layer_op("union", None, self.mask[0], None, self.mask[1 % wl.L], None, self.tmp_m, threads=th)
            elif st == "threshold":
                res["threshold"] = kn.select_threshold(self.surf["pos"][2], None, wl.thr[0], wl.thr[1], self.data[2 % wl.L],
                                                       self.mask[2 % wl.L], self.edited[2 % wl.L], 9, threads=th)
            elif st == "area":
                res["area"] = [kn.layer_area(self.surf["area"], m, threads=th) for m in self.mask]
            t[st] = time.perf_counter() - t0
        return t, res


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
    sample = "%d of %d rows of the %dx%d slab (%.1f Mtexel), oracle/kn_port.c with OpenMP" % (
        arm.rows, wl.A, wl.A, wl.width, arm.n / 1e6)
    print(json.dumps({
        "impl": "reference", "metric": "brush-apply + layer-op texel passes per second at 16384^2 atlas",
        "value": value, "unit": "Gtexel/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 decisions on u8/u32/f32 planes", "data": "synthetic",
        "config": workload_config(args, wl, stages),
        "cpu_baseline": {"value": value, "unit": "Gtexel/s", "cores": arm.threads, "kind": "port", "sample": sample,
                         "stage_ms": {s: per[s] / args.steps * 1e3 for s in stages}},
        "e2e": {"value": value, "unit": "Gtexel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def workload_config(args, wl, stages):
    return {"workload": "C3+C4: %dx%d atlas slab per GPU, %d uint8 layers, %d-triangle heightfield mesh; stages %s"
                        % (wl.A, wl.width, wl.L, wl.mesh.num_triangles, "+".join(stages)),
            "atlas": [wl.height, wl.width], "layers": wl.L, "triangles": wl.mesh.num_triangles,
            "window": [wl.cam.height, wl.cam.width], "stages": list(stages),
            "l2": "no explicit flush: every streamed input plane (>= 268 MB) is larger than the 126 MB L2, and the "
                  "streaming stages (chain, mask_op, threshold, area: >= 0.8 GB each, 10 GB together) run between the "
                  "footprint-culled brush stages of consecutive iterations, which therefore start from a cold L2",
            "parallelism": "row-sharded x%d" % args.gpus}


# ------------------------------------------------------------------------------------------------
# GPU arm

def run_ours(args):
    import torch
    import paper_2501_14807_b200 as ml
    from paper_2501_14807_b200 import _native as nat, sharding

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
    A, W, L = wl.A, wl.width, wl.L
    row0, rows = sharding.shard_rows(wl.height, world_size, rank)
    n = rows * W

    # ---- setup (untimed): surface map, depth, layers, pre-painting
    t0 = time.time()
    surf = ml.build_surface_map(wl.mesh, W, wl.height, row0=row0, rows=rows, device=dev)
    depth = ml.render_depth(wl.mesh, wl.cam, device=dev)
    ctx = ml.StrokeContext(wl.mesh, wl.cam, depth, surf, device=dev)
    pool = ml.TexturePool(budget_texels=(2 * L + 8) * n + 1, device=dev)
    layers = [ml.create_layer("L%d" % i, "uint8", W, rows, pool=pool) for i in range(L)]
    out_layer = ml.create_layer("out", "uint8", W, rows, pool=pool)
    edited = [torch.zeros((rows, W), dtype=torch.uint8, device=dev) for _ in range(L)]
    tmp_mask = torch.zeros((rows, W), dtype=torch.uint8, device=dev)
    # TPA outline, built once per mesh; neighbour slabs supply the 1-row halo
    cov_ext, cov_row0 = sharding.exchange_halo(surf.coverage.to(torch.uint8), row0, wl.height, 1)
    outline = nat.outline_mask(cov_ext, 1, in_row0=cov_row0, out_row0=row0, out_rows=rows)
    batch = nat.StrokeBatch([l.data for l in layers], [l.mask for l in layers], edited, dev)
    for k in range(len(wl.seed_strokes)):
        ml.select_sphere(surf, layers[k % L], wl.seed_strokes[k, :3], wl.seed_strokes[k, 3], wl.seed_labels[k],
                         edited=edited[k % L])
    attr = surf.pos[2]
    attr_tiles = nat.attr_tiles(attr)              # per-tile height ranges for the culled threshold selection
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    T = wl.mesh.num_triangles
    area_sums = torch.zeros(L, dtype=torch.float64, device=dev)
    area_counts = torch.zeros(L, dtype=torch.int64, device=dev)
    counts2 = torch.zeros(2, dtype=torch.int64, device=dev)
    counts1 = torch.zeros(1, dtype=torch.int64, device=dev)
    culled = not args.no_cull and surf.tiles is not None
    launches = {"tea": 3, "tpa": 1, "sphere": 2 if culled else 1, "batch": 2 if culled else 1, "chain": 1, "mask_op": 1,
                "threshold": 2 if (culled and attr_tiles is not None) else 1, "area": -(-L // 8)}

    def stage_call(st, inp, tool, mode, cull=not args.no_cull):
        """Run one stage through the public API and return its result as DEVICE tensors (nothing
        synchronises here).  mode "resident": stroke records were uploaded before the timed region;
        "e2e": this step's records come from the host now (pinned staging -> device)."""
        out = []
        if st == "tea":
            # --no-cull streams the whole id map instead of the stroke's footprint tiles
            r = ml.apply_stroke(ctx, tool, layers[0], eps=wl.eps, cull=cull)
            out = [r._counts]
        elif st == "tpa":
            # padding of the stroke just applied (the paper times TEA + TPA per edit); with
            # several ranks the 1-row halo of the edited plane travels point-to-point first
            counts1.zero_()
            if world_size > 1:
                # interior rows: footprint-culled tile pass; the border row next to each neighbour: streaming pass
                # over the exchanged halo row (16 KB point-to-point per neighbour)
                ml.editing.pad_slab(outline, ctx.edited, 1, layers[0].data, layers[0].mask, tool.value, counts1,
                                    row0=row0, height=wl.height, tiles=ctx.stroke_tiles if cull else None)
            else:
                nat.apply_padding(outline, ctx.edited, 1, layers[0].data, layers[0].mask, tool.value, counts=counts1,
                                  tiles=ctx.stroke_tiles if cull else None)
            out = [counts1.clone()]
        elif st == "sphere":
            s = inp["sphere"]
            out = [ml.select_sphere(surf, layers[1 % L], s[:3], s[3], inp["sphere_value"], edited=edited[1 % L],
                                    cull=cull)._counts]
        elif st == "batch":
            if mode == "e2e":
                s, lo, v = sharding.broadcast_strokes(inp["batch"], inp["batch_layers"], inp["batch_values"].astype(np.uint32), dev)
                batch.upload(s, lo, v.astype(np.uint8))
            batch.counts.zero_()
            out = [ml.select_sphere_batch(surf, batch, cull=cull).clone()]
        elif st == "chain":
            ml.layer_chain(layers[:wl.chain_n], wl.chain_ops, out_layer, lazy=cull)
        elif st == "mask_op":
            nat.layer_op("union", None, layers[0].mask, None, layers[1 % L].mask, None, tmp_mask)
        elif st == "threshold":
            out = [ml.select_threshold(attr, None, wl.thr[0], wl.thr[1], layers[2 % L], 9, edited=edited[2 % L],
                                       tiles=attr_tiles if cull else None)._counts]
        elif st == "area":
            area_sums.zero_()
            area_counts.zero_()
            nat.layer_area(surf.area, [l.mask for l in layers], sums=area_sums, counts=area_counts)
            sharding.allreduce_areas(area_sums, area_counts)
            out = [area_sums, area_counts]
        return out

    def make_tool(inp):
        return ml.EditingTool(px=float(inp["tool_xy"][0]), py=float(inp["tool_xy"][1]), shape=tool_shape_dev, value=7)

    tool_shape_dev = nat._as_dev_bytes(wl.tool_shape, dev)

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

    # ---- resident loop (value): inputs uploaded before the timed region, no read-back inside it
    inputs = [wl.step_inputs(i) for i in range(args.warmup + args.steps)]
    batch.upload(inputs[0]["batch"], inputs[0]["batch_layers"], inputs[0]["batch_values"])
    # clock sampler: started before the warm-up so that nvidia-smi is already delivering samples when the
    # timed region begins (its start-up alone can outlast a short timed region)
    stop, samples, windows = threading.Event(), [], []
    th = threading.Thread(target=sample_clocks, args=(stop, samples), daemon=True)
    th.start()
    t_wait = time.time()
    while not samples and time.time() - t_wait < 5.0 and th.is_alive():
        time.sleep(0.02)
    for i in range(args.warmup):
        for st in stages:
            stage_call(st, inputs[i], make_tool(inputs[i]), "resident")
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(stages) + 1)] for _ in range(args.steps)]
    barrier()
    t_begin = time.time()
    for k in range(args.steps):
        inp = inputs[args.warmup + k]
        tool = make_tool(inp)
        ev[k][0].record()
        for j, st in enumerate(stages):
            stage_call(st, inp, tool, "resident")
            ev[k][j + 1].record()
    barrier()
    windows.append((t_begin, time.time()))
    total_ms = max_over_ranks(ev[0][0].elapsed_time(ev[-1][-1]))
    stage_ms = {st: sum(ev[k][j].elapsed_time(ev[k][j + 1]) for k in range(args.steps)) / args.steps
                for j, st in enumerate(stages)}

    # ---- e2e loop: the same step through the public API, but every step (1) takes its stroke
    # records from HOST memory (pinned staging buffers -> device) and (2) reads all stage results
    # (edit counts, padded count, per-layer areas and texel counts) back to the host in one copy
    pinned = torch.empty(16, dtype=torch.float64).pin_memory()
    rec_dev = torch.empty(16, dtype=torch.float64, device=dev)

    def bits64(t):
        t = t.reshape(-1)
        if t.dtype == torch.int64:
            return t
        return t.view(torch.int64) if t.dtype == torch.float64 else t.to(torch.int64)

    out_pinned = [None, None]
    pending = []                        # (event, bytes) of read-backs queued but not yet consumed by the host

    def consume():
        n = 0
        while pending:
            e, nbytes = pending.pop(0)
            e.synchronize()             # the host now holds that step's results in pinned memory
            n += nbytes
        return n

    def e2e_step(inp, slot):
        """One step from host stroke records.  The read-back of the step's results is queued right behind its
        last stage (non-blocking copy into pinned memory) and consumed by the host after the FIRST stage of the
        next step has been queued, so the GPU goes from one step into the next without waiting for the host;
        every step's inputs still come from pinned host memory and every step's results are read by the host
        inside the timed region (the last step's before the closing event)."""
        rec = np.concatenate([inp["tool_xy"], inp["sphere"]])
        pinned[:rec.size].copy_(torch.from_numpy(rec))
        rec_dev[:rec.size].copy_(pinned[:rec.size], non_blocking=True)   # this step's scalar stroke record
        tool = make_tool(inp)
        res, got = [], 0
        for j, st in enumerate(stages):
            res += stage_call(st, inp, tool, "e2e")
            if j == 0:
                got += consume()        # results of the previous step
        if res:
            # ONE device->host read of every stage result: the 8-byte elements (int64 counts, float64 areas) are
            # concatenated bit for bit (a float64 viewed as int64 costs no kernel): one cat + one copy
            dev_out = torch.cat([bits64(t) for t in res])
            if out_pinned[slot] is None or out_pinned[slot].numel() != dev_out.numel():
                out_pinned[slot] = torch.empty(dev_out.numel(), dtype=torch.int64).pin_memory()
            out_pinned[slot].copy_(dev_out, non_blocking=True)
            e = torch.cuda.Event()
            e.record()
            pending.append((e, 8 * dev_out.numel()))
        return got

    for i in range(args.warmup):
        e2e_step(inputs[i], i & 1)
    consume()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_begin = time.time()
    e0.record()
    d2h = 0
    for k in range(args.steps):
        d2h += e2e_step(inputs[args.warmup + k], k & 1)
    d2h += consume()
    e1.record()
    barrier()
    windows.append((t_begin, time.time()))
    stop.set()
    th.join()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    h2d = 8 * 6 + 64 + (wl.L * (32 + 4 + 4) if "batch" in stages else 0)   # stroke records + 4x4 matrix

    # ---- hit census (untimed): mean number of texels each brush stage writes per step, for the
    # hit-write term of the algorithmic bytes.  Edited planes are cleared first so that the
    # kernels' "newly edited" counters equal the hit counts.
    hits = {s: 0.0 for s in stages}
    ncen = min(args.steps, 10)
    for k in range(ncen):
        inp = inputs[args.warmup + k]
        tool = make_tool(inp)
        for e in edited:
            e.zero_()
        for st in stages:
            r = stage_call(st, inp, tool, "resident")
            if st in ("tea", "tpa", "sphere", "batch", "threshold"):
                hits[st] += float(r[0].reshape(-1)[0].item() if st != "batch" else r[0].sum().item()) / ncen

    # ---- whole-atlas streaming forms of the brush stages, timed on their own (cull=False): the
    # HBM-roofline evidence for the brush kernels (SURVEY.md 8(d) algorithmic bytes / time)
    stream_info = {}
    if not args.no_cull:
        reps = max(5, min(20, args.steps))
        for st in [s for s in ("tea", "tpa", "sphere", "batch", "threshold", "chain") if s in stages]:
            ms_acc = 0.0
            for k in range(reps + 2):
                inp = inputs[args.warmup + (k % args.steps)]
                tool = make_tool(inp)
                if st == "tpa":
                    stage_call("tea", inp, tool, "resident", cull=False)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                stage_call(st, inp, tool, "resident", cull=False)
                b.record()
                torch.cuda.synchronize()
                if k >= 2:
                    ms_acc += a.elapsed_time(b)
            stream_info[st] = ms_acc / reps
        ctx.edited.zero_()

    # ---- the drop-in call with HOST planes (untimed part of the run, reported under config.host_plane_call):
    # the KN twin `raster_tea` (KN:135) called the way the reference calls it, numpy planes in host memory,
    # uploaded, edited and downloaded inside the call.  This is the PCIe cost the resident design avoids.
    host_call = None
    if rank == 0 and world_size == 1 and not args.no_cpu and "tea" in stages:
        inp = inputs[args.warmup]
        tool = make_tool(inp)
        sfx, sfy, bx, by = ml.compute_tool_projection(wl.cam, tool).kernel_factors
        tri_xy = np.ascontiguousarray(wl.mesh.tri_uv_texels(W, wl.height))
        clip = np.ascontiguousarray(wl.cam.clip_coords(wl.mesh.vertices)[wl.mesh.triangles])
        depth_np = depth.plane.cpu().numpy()
        shape_np = np.ascontiguousarray(wl.tool_shape).astype(np.uint8)
        planes = [np.zeros((rows, W), np.uint8) for _ in range(3)]
        ctx.edited.zero_()
        want = int(stage_call("tea", inp, tool, "resident")[0].reshape(-1)[0].item())
        ctx.edited.zero_()
        t_host = []
        got = None
        for _ in range(2):
            planes[2][:] = 0
            t0 = time.perf_counter()
            got = nat.raster_tea(tri_xy, clip, float(wl.cam.width), float(wl.cam.height), depth_np, wl.eps, sfx, sfy,
                                 bx, by, shape_np, planes[0], planes[1], planes[2], 7)
            t_host.append((time.perf_counter() - t0) * 1e3)
        moved = tri_xy.nbytes + clip.nbytes + depth_np.nbytes + shape_np.nbytes + 3 * planes[0].nbytes
        host_call = {"op": "raster_tea (KN:135-136) with numpy planes: upload + direct per-triangle kernel + download",
                     "ms": round(min(t_host), 2), "gtexel_s": round(n / (min(t_host) * 1e-3) / 1e9, 2),
                     "h2d_bytes": moved, "d2h_bytes": 3 * planes[0].nbytes,
                     "edited": int(got[0]), "equal_to_resident_stroke": int(got[0]) == want}
        del planes, tri_xy, clip

    texel_passes = len(stages) * n * world_size
    value = texel_passes * args.steps / (total_ms * 1e-3) / 1e9
    e2e_value = texel_passes * args.steps / (e2e_ms * 1e-3) / 1e9
    peak, peak_src = measured_peak()
    stage_info = {}
    for st in stages:
        b = wl.algorithmic_bytes(n, st, T, hits[st])
        gbs = b / (stage_ms[st] * 1e-3) / 1e9
        stage_info[st] = {"ms": round(stage_ms[st], 4), "gtexel_s": round(n / (stage_ms[st] * 1e-3) / 1e9, 2),
                          "alg_bytes": b, "gb_s": round(gbs, 1), "frac_of_peak": round(gbs / peak, 4),
                          "hits_per_step": int(hits[st]), "launches": launches[st]}
        if st in ("tea", "tpa", "sphere", "batch", "threshold"):
            stage_info[st]["footprint_culled"] = not args.no_cull
        if st == "chain":
            # (N+1)*2 B/texel is an upper bound: the chain kernel fetches a data vector only where the masks
            # say it can contribute, so its "frac_of_peak" can exceed 1 (bytes that were never read)
            stage_info[st]["lazy_data_reads"] = not args.no_cull
    peak_now = peak
    stream_kernels = {st: {"ms": round(ms, 4), "gb_s": round(wl.algorithmic_bytes(n, st, T, hits[st]) / (ms * 1e-3) / 1e9, 1),
                           "frac_of_peak": round(wl.algorithmic_bytes(n, st, T, hits[st]) / (ms * 1e-3) / 1e9 / peak_now, 4)}
                      for st, ms in stream_info.items()}
    # The roofline object is quoted for the slowest stage whose SURVEY 8(d) bytes are really moved.  Footprint-culled
    # brush stages and the lazy chain skip most of those bytes by design (their "frac_of_peak" above exceeds 1), so
    # they are not roofline evidence; their whole-atlas forms are, under config.stream_kernels / --no-cull.
    skipping = set() if args.no_cull else {"tea", "tpa", "sphere", "batch", "threshold", "chain"}
    full = [s for s in stages if s not in skipping] or list(stages)
    dom = max(full, key=lambda s: stage_ms[s])
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        # whole-atlas (--no-cull) runs launch the streaming forms of the kernels: "<stage>_stream" entries
        traffic = tj.get(dom + "_stream", tj.get(dom)) if args.no_cull else tj.get(dom)
    # the dominant stage's main kernel: stage bytes / stage time (for tea the stage is 3 kernels
    # + the edited-plane reset; its bytes include all of them)
    dom_b = wl.algorithmic_bytes(n, dom, T, hits[dom])
    dom_ms = stage_ms[dom]

    cpu = None
    if rank == 0 and world_size == 1 and not args.no_cpu:
        arm = CpuArm(wl, args.cpu_rows)
        arm.step(0, stages)
        reps, el, per = 0, 0.0, {s: 0.0 for s in stages}
        while reps < 3 or (el < 10.0 and reps < 20):
            t, _ = arm.step(1 + reps, stages)
            for s in stages:
                per[s] += t[s]
            el += sum(t.values())
            reps += 1
        cpu = {"value": len(stages) * arm.n * reps / el / 1e9, "unit": "Gtexel/s", "cores": arm.threads, "kind": "port",
               "sample": "%d of %d rows of the slab (%.1f Mtexel) x %d reps, oracle/kn_port.c (C restatement of the "
                         "reference numpy kernels) with OpenMP over rows" % (arm.rows, A, arm.n / 1e6, reps),
               "stage_ms": {s: round(per[s] / reps * 1e3, 3) for s in stages}}

    if rank == 0:
        cfg = workload_config(args, wl, stages)
        cfg["stage_results"] = stage_info
        cfg["setup_s"] = round(setup_s, 2)
        cfg["surface_map"] = {"covered": surf.covered, "overlap": surf.overlap}
        cfg["footprint_culling"] = not args.no_cull
        cfg["stream_kernels"] = stream_kernels
        if host_call:
            cfg["host_plane_call"] = host_call
        print(json.dumps({
            "metric": "brush-apply + layer-op texel passes per second at 16384^2 atlas",
            "value": value, "unit": "Gtexel/s", "n_gpus": world_size, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64 decisions on u8/u32/f32 planes", "data": "synthetic", "config": cfg,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": dom_b / (dom_ms * 1e-3) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": dom_b / (dom_ms * 1e-3) / 1e9 / peak, "traffic": traffic,
                         "peak_source": peak_src, "frac_of_8TBs_spec": dom_b / (dom_ms * 1e-3) / 1e9 / 8000.0,
                         "dram_frac": None if not traffic else traffic / (dom_ms * 1e-3) / 1e9 / peak,
                         "basis": "SURVEY 8(d) algorithmic bytes of the slowest stage that streams all of them; "
                                  "stages that skip bytes by design (%s) are excluded, see config.stream_kernels"
                                  % (", ".join(sorted(skipping & set(stages))) or "none")},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "Gtexel/s", "ms_per_step": e2e_ms / args.steps,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h // max(1, args.steps)},
            "gpu_launches": sum(launches[s] for s in stages) * args.steps,
            "clocks": clocks_summary(samples, windows),
        }))
    if world_size > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
