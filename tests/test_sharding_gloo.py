"""world_size-2 tests of the multi-GPU host logic on CPU tensors with the gloo backend:
stroke broadcast, area all-reduce, halo exchange, and "row slabs concatenate to the full plane"
with the oracle standing in for the per-rank kernels (the test may use the oracle; the product
never does)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import kn
from paper_2501_14807_b200 import sharding, synth


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world_size, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    try:
        assert sharding.world() == (rank, world_size)
        # ---- stroke broadcast: only rank 0 knows the strokes
        mesh = synth.icosphere_mesh(2)
        if rank == 0:
            strokes, labels = synth.sphere_strokes(mesh, 5, seed=3, rmin_frac=0.1, rmax_frac=0.3)
            layer_of = np.array([0, 1, 0, 1, 0], np.int32)
            vals = labels.astype(np.uint32)
        else:
            strokes, layer_of, vals = np.zeros((0, 4)), np.zeros(0, np.int32), np.zeros(0, np.uint32)
        s, lo, v = sharding.broadcast_strokes(strokes, layer_of, vals, "cpu")
        want_s, want_l = synth.sphere_strokes(mesh, 5, seed=3, rmin_frac=0.1, rmax_frac=0.3)
        assert np.array_equal(s, want_s) and np.array_equal(v, want_l.astype(np.uint32))
        assert lo.tolist() == [0, 1, 0, 1, 0]

        # ---- each rank computes its row slab (oracle as the local kernel), then all-reduces areas
        A = 96
        r0, rows = sharding.shard_rows(A, world_size, rank)
        surf = kn.surface_map(mesh.tri_uv_texels(A, A), mesh.tri_pos(), mesh.tri_nrm(), A, A, rows=(r0, r0 + rows))
        data = [np.zeros((rows, A), np.uint8) for _ in range(2)]
        mask = [np.zeros((rows, A), np.uint8) for _ in range(2)]
        edited = [np.zeros((rows, A), np.uint8) for _ in range(2)]
        counts = torch.zeros(2, dtype=torch.int64)
        for k in range(len(s)):
            L = int(lo[k])
            counts[L] += kn.select_sphere(surf["pos"], s[k, :3], s[k, 3], data[L], mask[L], edited[L], int(v[k]))
        sums = torch.tensor([kn.layer_area(surf["area"], m)[0] for m in mask], dtype=torch.float64)
        texels = torch.tensor([kn.layer_area(surf["area"], m)[1] for m in mask], dtype=torch.int64)
        # the per-step form: raw 8-byte slots, one all-gather, summed in rank order on every rank
        slots = torch.cat([sums.view(torch.int64), texels])
        sharding.AreaReducer(2, "cpu")(slots)
        sharding.allreduce_areas(sums, texels)
        sharding.allreduce_counts(counts)
        assert torch.equal(slots[2:], texels)
        assert torch.allclose(slots[:2].view(torch.float64), sums, rtol=1e-15, atol=0.0)
        # a batch larger than the broadcast buffer travels in several rounds
        if rank == 0:
            big = np.arange(44, dtype=np.float64).reshape(11, 4)
            got = sharding.broadcast_strokes(big, np.arange(11, dtype=np.int32), np.arange(11, dtype=np.uint32) + 7, "cpu", capacity=4)
        else:
            got = sharding.broadcast_strokes(np.zeros((0, 4)), np.zeros(0, np.int32), np.zeros(0, np.uint32), "cpu", capacity=4)
        assert np.array_equal(got[0], np.arange(44, dtype=np.float64).reshape(11, 4))
        assert got[1].tolist() == list(range(11)) and got[2].tolist() == [k + 7 for k in range(11)]

        # ---- the set-up vote: true only if every rank says so (a local failure takes all ranks to the fallback)
        assert sharding.agree(True) is True
        assert sharding.agree(rank != 1) is False
        assert sharding.agree(False) is False

        # ---- halo exchange of a byte plane for a radius-2 stencil
        cov = torch.from_numpy((surf["tri_id"] >= 0).astype(np.uint8))
        ext, ext_row0 = sharding.exchange_halo(cov, r0, A, 2)
        in0, in_rows = sharding.halo_bounds(r0, rows, A, 2)
        assert ext_row0 == in0 and ext.shape[0] == in_rows
        # the per-stroke form: only the received rows, no extended copy of the slab
        up, dn = sharding.exchange_halo(cov, r0, A, 2, parts=True)
        k = r0 - ext_row0
        assert (up is None) == (k == 0) and (dn is None) == (ext.shape[0] == k + rows)
        if up is not None:
            assert torch.equal(up, ext[:k])
        if dn is not None:
            assert torch.equal(dn, ext[k + rows:])
        # the stroke-path form: the halo rows land in the spare rows of the rank's own plane (no concatenation)
        margin = 4
        buf = torch.zeros((rows + 2 * margin, A), dtype=torch.uint8)
        buf[margin:margin + rows] = cov
        up_n, dn_n = sharding.exchange_halo_into(buf, margin, rows, r0, A, 2)
        assert (up_n, dn_n) == (0 if up is None else up.shape[0], 0 if dn is None else dn.shape[0])
        assert torch.equal(buf[margin - up_n:margin + rows + dn_n], ext)
        assert not bool(buf[:margin - up_n].any()) and not bool(buf[margin + rows + dn_n:].any())
        np.savez(os.path.join(out_dir, "rank%d.npz" % rank), data0=data[0], data1=data[1], mask0=mask[0], mask1=mask[1],
                 sums=sums.numpy(), texels=texels.numpy(), counts=counts.numpy(), ext=ext.numpy(), ext_row0=ext_row0,
                 r0=r0, rows=rows)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_two_rank_row_sharding_equals_single_rank(tmp_path):
    ws = 2
    mp.spawn(_worker, args=(ws, _free_port(), str(tmp_path)), nprocs=ws, join=True)
    parts = [np.load(tmp_path / ("rank%d.npz" % r)) for r in range(ws)]
    # single-process reference over the full atlas
    mesh = synth.icosphere_mesh(2)
    A = 96
    surf = kn.surface_map(mesh.tri_uv_texels(A, A), mesh.tri_pos(), mesh.tri_nrm(), A, A)
    strokes, labels = synth.sphere_strokes(mesh, 5, seed=3, rmin_frac=0.1, rmax_frac=0.3)
    data = [np.zeros((A, A), np.uint8) for _ in range(2)]
    mask = [np.zeros((A, A), np.uint8) for _ in range(2)]
    edited = [np.zeros((A, A), np.uint8) for _ in range(2)]
    counts = [0, 0]
    for k, L in enumerate([0, 1, 0, 1, 0]):
        counts[L] += kn.select_sphere(surf["pos"], strokes[k, :3], strokes[k, 3], data[L], mask[L], edited[L], int(labels[k]))
    for L in range(2):
        assert np.array_equal(np.concatenate([p["data%d" % L] for p in parts]), data[L])
        assert np.array_equal(np.concatenate([p["mask%d" % L] for p in parts]), mask[L])
        a, c = kn.layer_area(surf["area"], mask[L])
        for p in parts:                                   # every rank holds the reduced totals
            assert abs(p["sums"][L] - a) <= 1e-12 * max(a, 1e-300) and p["texels"][L] == c
            assert p["counts"][L] == counts[L]
    cov = (surf["tri_id"] >= 0).astype(np.uint8)
    for p in parts:
        e0 = int(p["ext_row0"])
        assert np.array_equal(p["ext"], cov[e0:e0 + p["ext"].shape[0]])
    assert sum(int(p["rows"]) for p in parts) == A


# ---- per-stroke TPA on row slabs: editing.pad_slab with a real gloo halo exchange --------------------

_CALLS = []


def _oracle_apply_padding(outline, edited, radius, data, mask, value, *, in_row0=0, out_row0=None, counts=None,
                          tiles=None, row_range=None):
    """Stand-in for _native.apply_padding on CPU tensors (the test may use the oracle; the product never
    does): same arguments, the oracle's padding over the given input window, restricted to `row_range`."""
    out_row0 = in_row0 if out_row0 is None else out_row0
    rows, w = outline.shape
    _CALLS.append("interior" if row_range is not None else "border")
    lo, hi = (0, rows) if row_range is None else row_range
    if hi <= lo:
        return
    # input window as a plane whose row 0 is global row in_row0; outputs start at global row out_row0
    ed = edited.numpy()
    off = out_row0 - in_row0
    # pad the window so that the oracle sees [out_row0 - radius, out_row0 + rows + radius)
    full = np.zeros((rows + 2 * radius, w), np.uint8)
    for r in range(rows + 2 * radius):
        src = off - radius + r
        if 0 <= src < ed.shape[0]:
            full[r] = ed[src]
    o = np.zeros_like(full)
    o[radius + lo:radius + hi] = outline.numpy()[lo:hi]
    d = np.zeros_like(full)
    m = np.zeros_like(full)
    d[radius:radius + rows] = data.numpy()
    m[radius:radius + rows] = mask.numpy()
    n = kn.padding(o, full, radius, d, m, value)
    data.copy_(torch.from_numpy(d[radius:radius + rows]))
    mask.copy_(torch.from_numpy(m[radius:radius + rows]))
    counts += n


def _pad_worker(rank, world_size, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    try:
        from paper_2501_14807_b200 import _native, editing
        _native.apply_padding = _oracle_apply_padding                     # no GPU in this test
        H, W, radius = 96, 128, 2
        rng = np.random.default_rng(5)
        outline = (rng.random((H, W)) < 0.3).astype(np.uint8)
        edited = np.zeros((H, W), np.uint8)
        edited[28:36, 20:90] = 1                                           # straddles the 32-row slab border
        edited[60:66, 5:40] = 1                                            # and the second one
        edited[rng.random((H, W)) < 0.01] = 1
        r0, rows = sharding.shard_rows(H, world_size, rank)
        data = torch.zeros((rows, W), dtype=torch.uint8)
        mask = torch.zeros((rows, W), dtype=torch.uint8)
        counts = torch.zeros(1, dtype=torch.int64)
        editing.pad_slab(torch.from_numpy(outline[r0:r0 + rows].copy()), torch.from_numpy(edited[r0:r0 + rows].copy()),
                         radius, data, mask, 7, counts, row0=r0, height=H, tiles=torch.zeros(1, dtype=torch.int32))
        # the decomposition under test really ran: one interior pass + one border pass per neighbour
        assert _CALLS.count("interior") == 1 and _CALLS.count("border") == (rank > 0) + (rank < world_size - 1), _CALLS
        # same stroke through the allocation-free form: the edited plane carries spare rows, the halo lands in them
        margin = 4
        buf = torch.zeros((rows + 2 * margin, W), dtype=torch.uint8)
        buf[margin:margin + rows] = torch.from_numpy(edited[r0:r0 + rows].copy())
        data2 = torch.zeros((rows, W), dtype=torch.uint8)
        mask2 = torch.zeros((rows, W), dtype=torch.uint8)
        counts2 = torch.zeros(1, dtype=torch.int64)
        del _CALLS[:]
        editing.pad_slab(torch.from_numpy(outline[r0:r0 + rows].copy()), buf[margin:margin + rows], radius, data2, mask2, 7,
                         counts2, row0=r0, height=H, tiles=torch.zeros(1, dtype=torch.int32), ext=(buf, margin))
        assert _CALLS.count("interior") == 1 and _CALLS.count("border") == (rank > 0) + (rank < world_size - 1), _CALLS
        assert torch.equal(data2, data) and torch.equal(mask2, mask) and int(counts2) == int(counts)
        sharding.allreduce_counts(counts)
        np.savez(os.path.join(out_dir, "pad%d.npz" % rank), data=data.numpy(), mask=mask.numpy(), count=counts.numpy(),
                 outline=outline, edited=edited)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_three_rank_slab_padding_equals_whole_plane(tmp_path):
    """editing.pad_slab on three ranks (gloo, CPU tensors, the oracle standing in for the padding kernels): the
    interior / border-row decomposition with the exchanged halo rows pads exactly the texels the whole-plane
    pass pads, and counts every one once."""
    ws = 3
    mp.spawn(_pad_worker, args=(ws, _free_port(), str(tmp_path)), nprocs=ws, join=True)
    parts = [np.load(tmp_path / ("pad%d.npz" % r)) for r in range(ws)]
    outline, edited = parts[0]["outline"], parts[0]["edited"]
    data, mask = np.zeros_like(outline), np.zeros_like(outline)
    want = kn.padding(outline, edited, 2, data, mask, 7)
    assert want > 0 and all(int(p["count"][0]) == want for p in parts)
    assert np.array_equal(np.concatenate([p["data"] for p in parts]), data)
    assert np.array_equal(np.concatenate([p["mask"] for p in parts]), mask)
