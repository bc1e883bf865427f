#!/usr/bin/env python
"""Surface-map build of ONE row slab of BASELINE config 5 (32768^2 atlas, 9,999,392 triangles): device time of the
whole build per slab count, for the launch list (`ncu --metrics gpu__time_duration.sum ... python tools/slab_build_prof.py 8`).

    python tools/slab_build_prof.py [slabs ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2501_14807_b200 as ml
    from paper_2501_14807_b200 import synth
    A = 32768
    mesh = synth.heightfield_mesh(2236, margin=0.01)
    for ns in [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]:
        rows = A // ns
        row0 = (ns // 2) * rows if ns > 1 else 0
        ts = []
        for rep in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            surf = ml.build_surface_map(mesh, A, A, row0=row0, rows=rows)
            e1.record()
            torch.cuda.synchronize()
            ts.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
            cov = surf.covered
            del surf
            torch.cuda.empty_cache()
        print("slabs %d: rows %d from %d: device %.2f ms (wall %.0f ms), covered %d" % (ns, rows, row0, min(t[0] for t in ts), min(t[1] for t in ts), cov), flush=True)


if __name__ == "__main__":
    main()
