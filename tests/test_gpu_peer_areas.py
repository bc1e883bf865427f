"""The fused cross-rank area reduction (sharding.PeerAreaReducer / ml_layer_area_peers): every rank's reduction kernel
adds its partials with system-scope atomics straight into every rank's result row over IPC-mapped peer memory, one
thread signals / awaits the arrival slots -- no collective call.  Exercised here with TWO processes: one GPU each
when the box has two (NVLink peer atomics), else sharing cuda:0 (CUDA IPC works between processes on one device; the
round's boxes have one GPU): global sums and counts
on both ranks == the whole-plane values, over more steps than the row ring holds (recycling), layer counts that
need one and several launch groups."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, L, steps, out_dir):
    import torch
    import torch.distributed as dist
    from paper_2501_14807_b200 import _native as nat, sharding
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    # one GPU per rank when the box has them (real NVLink peer atomics), else both ranks share cuda:0 (IPC on one device)
    index = rank if torch.cuda.device_count() >= ws else 0
    torch.cuda.set_device(index)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        dev = torch.device("cuda", index)
        H, W = 512, 640                                       # whole plane; rank r owns rows shard_rows(H, ws, r)
        rng = np.random.default_rng(99)
        area = rng.random((H, W)).astype(np.float32)
        base = [(rng.random((H, W)) < 0.1 + 0.05 * (k % 7)).astype(np.uint8) for k in range(L)]
        r0, rows = sharding.shard_rows(H, ws, rank)
        d_area = torch.from_numpy(area[r0:r0 + rows].copy()).to(dev)
        try:
            red = sharding.PeerAreaReducer(L, dev)
        except Exception as exc:                              # CUDA IPC not permitted in this container: nothing to test
            with open(os.path.join(out_dir, "skip%d" % rank), "w") as f:
                f.write(repr(exc))
            return
        assert red.self_test()
        dist.barrier()
        out = torch.zeros(2 * L, dtype=torch.int64, device=dev)
        worst = 0.0
        for step in range(steps):
            shift = 3 * step                                  # different masks every step (rolled columns)
            full = [np.roll(m, shift, axis=1) for m in base]
            masks = [torch.from_numpy(np.ascontiguousarray(m[r0:r0 + rows])).to(dev) for m in full]
            red.reduce(step, d_area, masks, out)
            got = out.cpu()
            sums = got[:L].view(torch.float64).numpy()
            cnts = got[L:].numpy()
            want_s = np.array([(area.astype(np.float64) * (m != 0)).sum() for m in full])
            want_c = np.array([(m != 0).sum() for m in full])
            assert np.array_equal(cnts, want_c), (rank, step, cnts, want_c)
            worst = max(worst, float(np.max(np.abs(sums - want_s) / want_s)))
        red.check()
        assert worst <= 1e-12
        dist.barrier()
        red.close()
        with open(os.path.join(out_dir, "ok%d" % rank), "w") as f:
            f.write("%g" % worst)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("L,steps", [(3, 40), (8, 20), (13, 10)])
def test_two_ranks_on_one_gpu_sum_into_each_others_rows(tmp_path, L, steps):
    import torch.multiprocessing as mp
    ws = 2
    mp.spawn(_worker, args=(ws, _free_port(), L, steps, str(tmp_path)), nprocs=ws, join=True)
    if any(os.path.exists(tmp_path / ("skip%d" % r)) for r in range(ws)):
        pytest.skip("CUDA IPC unavailable here: " + open([p for p in tmp_path.iterdir() if p.name.startswith("skip")][0]).read())
    assert all(os.path.exists(tmp_path / ("ok%d" % r)) for r in range(ws))
