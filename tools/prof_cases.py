#!/usr/bin/env python
"""One launch of each tuning case, for ncu captures (no warm-up, no repetition):

    ncu --set full --clock-control none --import-source on -k regex:"resolve|raster_warp" \
        -o gpurun_out/x python tools/prof_cases.py surface

Cases: surface (16384^2 surface-map build of the C2 mesh), sphere (few hits, 50% hits),
threshold (coherent 50%, noise 20%), tpa (outline build + padding), area (L=1, L=4),
octree (only when named: depth-12 octree of the C2 mesh + one r=200 ray-cast edit)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_14807_b200 import _native as nat, synth  # noqa: E402


def main():
    want = set(sys.argv[1:]) or {"surface", "sphere", "threshold", "tpa", "area"}
    if "octree" in want:
        import paper_2501_14807_b200 as ml
        from paper_2501_14807_b200 import bench
        mesh = bench.make_mesh("terrain:707")
        cam = bench.make_camera("terrain:707", (1024, 1024))
        tree = ml.build_octree(mesh, 12)
        layer = ml.create_octree_layer(tree)
        tool = ml.EditingTool(px=512.0, py=512.0, shape=synth.circle_shape(200), value=7)
        ml.octree_edit(tree, layer, mesh, cam, tool)
        torch.cuda.synchronize()
        del tree, layer
        torch.cuda.empty_cache()
        want.discard("octree")
        if not want:
            return
    N = int(os.environ.get("PROF_N", "16384"))
    n = N * N
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(1)
    if "surface" in want:
        mesh = synth.heightfield_mesh(707, margin=0.01)
        xy = torch.from_numpy(mesh.tri_uv_texels(N, N)).to(dev)
        P, Nn = torch.from_numpy(mesh.tri_pos()).to(dev), torch.from_numpy(mesh.tri_nrm()).to(dev)
        nat.surface_map(xy, P, Nn, N, N)
        torch.cuda.synchronize()
        del xy, P, Nn
        torch.cuda.empty_cache()
    data = torch.zeros((N, N), dtype=torch.uint8, device=dev)
    mask = torch.zeros((N, N), dtype=torch.uint8, device=dev)
    edited = torch.zeros((N, N), dtype=torch.uint8, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    if "sphere" in want:
        pos = torch.rand((3, N, N), device=dev, generator=g)
        nat.select_sphere(pos, (0.5, 0.5, 0.5), 0.05, data, mask, edited, 3, counts=cnt)
        nat.select_sphere(pos, (0.5, 0.5, 0.5), 0.62, data, mask, edited, 3, counts=cnt)
        torch.cuda.synchronize()
        del pos
    if "threshold" in want:
        yy, xx = torch.meshgrid(torch.linspace(0, 6, N, device=dev), torch.linspace(0, 6, N, device=dev), indexing="ij")
        attr = (torch.sin(xx) * torch.cos(yy)).contiguous()
        del yy, xx
        edited.zero_()
        nat.select_threshold(attr, None, -0.5, 0.5, data, mask, edited, 3, counts=cnt)
        noise = torch.rand((N, N), device=dev, generator=g)
        edited.zero_()
        nat.select_threshold(noise, None, 0.0, 0.2, data, mask, edited, 3, counts=cnt)
        torch.cuda.synchronize()
        del attr, noise
    if "tpa" in want:
        cov = torch.zeros((N, N), dtype=torch.uint8, device=dev)
        cov[N // 100: N - N // 100, N // 100: N - N // 100] = 1
        ring = nat.outline_mask(cov, 1)
        edited.zero_()
        edited[N // 2 - 500: N // 2 + 500, N // 2 - 500: N // 2 + 500] = 1
        nat.apply_padding(ring, edited, 1, data, mask, 3, counts=cnt)
        torch.cuda.synchronize()
        del cov, ring
    if "area" in want:
        area = torch.rand((N, N), device=dev, generator=g)
        m2 = (torch.rand((N, N), device=dev, generator=g) < 0.3).to(torch.uint8)
        masks = [m2, mask, edited, data]
        nat.layer_area(area, masks[:1], sums=torch.zeros(1, dtype=torch.float64, device=dev),
                       counts=torch.zeros(1, dtype=torch.int64, device=dev))
        nat.layer_area(area, masks, sums=torch.zeros(4, dtype=torch.float64, device=dev),
                       counts=torch.zeros(4, dtype=torch.int64, device=dev))
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
