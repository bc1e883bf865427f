#!/usr/bin/env python
"""Turn ncu output into the small, committed artefacts under profiles/.

    python tools/profile_summary.py launches  gpurun_out/launches.csv  profiles/r1_launches.md
    python tools/profile_summary.py full      gpurun_out/prof.ncu-rep  profiles/r1_ncu_full.md  profiles/traffic.json

`launches` aggregates the `--metrics gpu__time_duration.sum` launch list per kernel (count, mean,
share of GPU time).  `full` extracts the roofline-relevant metrics of a `--set full` capture
(read here with `ncu -i ... --page raw --csv`) and writes per-stage DRAM traffic per launch."""
import collections
import csv
import json
import subprocess
import sys

# kernel-name substring -> the bench stages it belongs to ("<stage>" = default path, "<stage>_stream" = whole-atlas
# form).  traffic.json sums ONE launch of every kernel of a stage (classification + main + evaluation kernels).
STAGE_OF = (("chain_lazy_kernel", ("chain",)), ("chain_kernel", ("chain_stream",)), ("binary_kernel", ("mask_op",)),
            ("sphere_batch_tiles_kernel", ("batch",)), ("sphere_batch_kernel", ("batch_stream",)),
            ("sphere_tiles_kernel", ("sphere",)), ("sphere_kernel", ("sphere_stream",)),
            ("tile_classify_kernel", ("sphere", "batch")),
            ("threshold_tiles_kernel", ("threshold",)), ("threshold_tiles_vec_kernel", ("threshold",)), ("range_classify_kernel", ("threshold",)),
            ("threshold_bulk_kernel", ("threshold_stream",)), ("threshold_vec_kernel", ("threshold_stream",)),
            ("threshold_kernel", ("threshold_stream",)),
            ("area_bulk_kernel", ("area",)), ("area_kernel", ("area",)),
            ("tea_eval_kernel", ("tea", "tea_stream")), ("tea_classify", ("tea", "tea_stream")),
            ("tea_tile_kernel", ("tea",)), ("tea_stream_bulk_kernel", ("tea_stream",)), ("tea_stream_kernel", ("tea_stream",)),
            ("padding_tile_kernel", ("tpa",)), ("padding_bulk_kernel", ("tpa_stream",)), ("padding_stream_kernel", ("tpa_stream",)))

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm %peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("smsp__inst_executed.sum", "warp insts"),
]


def short(name):
    name = name.replace("void ", "").replace("<unnamed>::", "")
    return name.split("(")[0][:60]


def launches(src, dst):
    rows = list(csv.reader(open(src)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    kn, mv, mu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in data:
        if len(r) <= mv:
            continue
        v = float(r[mv].replace(",", ""))
        if r[mu] in ("us", "usecond"):
            v *= 1e3
        elif r[mu] in ("ms", "msecond"):
            v *= 1e6
        a = agg.setdefault(short(r[kn]), [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    with open(dst, "w") as f:
        f.write("# ncu launch list (gpu__time_duration.sum, --clock-control none), aggregated per kernel\n\n")
        f.write("Source: `%s`.  Per-launch times are cold-cache and serialised by ncu: compare SHARES.\n\n" % src)
        f.write("| kernel | launches | mean us | share of GPU time |\n|---|---|---|---|\n")
        for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write("| `%s` | %d | %.1f | %.1f%% |\n" % (k, c, t / c / 1e3, 100 * t / tot))
    print("wrote", dst)


def _raw_csv(src):
    if src.endswith(".csv"):        # already exported on the GPU box: ncu -i x.ncu-rep --page raw --csv > x.csv
        return open(src).read()
    return subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout


def full(srcs, dst, traffic_dst=None):
    """``srcs``: one report / raw CSV or several separated by commas (each keeps its own unit row)."""
    seen, traffic = set(), {}
    with open(dst, "w") as f:
        f.write("# ncu --set full --clock-control none: key metrics per kernel (first captured launch of each)\n\n")
        f.write("Source reports: `%s` (not committed; regenerate with the commands in profiles/README.md).\n\n" % srcs)
        for src in srcs.split(","):
            rows = list(csv.reader(_raw_csv(src).splitlines()))
            hdr, units, data = rows[0], rows[1], rows[2:]
            kn = hdr.index("Kernel Name")
            stall = [(i, h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                     for i, h in enumerate(hdr) if "smsp__average_warps_issue_stalled" in h and h.endswith("_per_issue_active.ratio")]

            def tobytes(r, m):
                i = hdr.index(m)
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[i]]
                return float(r[i].replace(",", "")) * scale
            for r in data:
                name = short(r[kn])
                if name in seen:
                    continue
                seen.add(name)
                f.write("## `%s`\n\n| metric | value |\n|---|---|\n" % name)
                for m, label in METRICS:
                    if m in hdr:
                        i = hdr.index(m)
                        f.write("| %s | %s %s |\n" % (label, r[i], units[i]))
                top = sorted(((float(r[i]), h) for i, h in stall if r[i]), reverse=True)[:4]
                f.write("| top stalls (warps per issue) | %s |\n\n" % ", ".join("%s %.2f" % (h, v) for v, h in top))
                for key, stages in STAGE_OF:
                    if key in name and "dram__bytes_read.sum" in hdr:
                        for stage in stages:
                            traffic[stage] = traffic.get(stage, 0.0) + tobytes(r, "dram__bytes_read.sum") + tobytes(r, "dram__bytes_write.sum")
                        break
    print("wrote", dst)
    if traffic_dst:
        # the capture is the default bench workload: 16384^2 texels, 8 layers (bench.py scales by texels for other sizes)
        traffic["_texels"] = 16384 * 16384
        traffic["_layers"] = 8
        json.dump(traffic, open(traffic_dst, "w"), indent=1, sort_keys=True)
        print("wrote", traffic_dst, traffic)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
