"""Row sharding of the atlas across the GPUs of one node.

Every hot kernel is independent per texel, so rank r owns the row slab [row0, row0+rows) of every
plane (surface map and all layers) and no data-path collective exists.  The only exchanges are
  * ``broadcast_strokes``: rank 0's stroke records (a few dozen bytes each; the paper's "64 bytes
    per stroke") -> all ranks, one broadcast per batch, and
  * ``allreduce_areas`` : per-layer partial area sums (float64) and texel counts (int64), one
    all-reduce for all layers.
Both are latency-bound scalars over NCCL/NVLink; with world_size == 1 they are no-ops.  The
stencil ops (outline / padding) need ``radius`` halo rows from the neighbouring slabs:
``exchange_halo`` does that with two point-to-point copies.

One process per GPU (torchrun); the same code runs on CPU tensors with the gloo backend, which
is how the host logic is tested without GPUs.
"""
import numpy as np


def _dist():
    import torch.distributed as dist
    return dist


def world():
    """(rank, world_size) of the default process group, (0, 1) when not initialised."""
    dist = _dist()
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_rows(height, world_size, rank):
    """Contiguous, balanced row slab of rank ``rank``: returns (row0, rows).  Slabs tile
    [0, height) exactly; the first ``height % world_size`` ranks get one extra row."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad rank / world size")
    base, extra = divmod(int(height), int(world_size))
    row0 = rank * base + min(rank, extra)
    return row0, base + (1 if rank < extra else 0)


def all_slabs(height, world_size):
    return [shard_rows(height, world_size, r) for r in range(world_size)]


def broadcast_strokes(strokes, layer_of, values, device, src=0, capacity=256):
    """Host-facing form: rank ``src`` supplies numpy arrays (strokes (K,4) f64, layer_of (K,) i32, values
    (K,) u32 bit patterns); every rank returns the same three numpy arrays.  ONE broadcast of a fixed
    (capacity+1, 6) float64 buffer whose first row carries K (batches larger than ``capacity`` go in several
    rounds).  Returning numpy means a read-back on the receivers; the per-step device path is
    ``broadcast_batch``, which has none."""
    import torch
    dist = _dist()
    rank, ws = world()
    if ws == 1:
        return strokes, layer_of, values
    outs, start = [], 0
    while True:
        buf = torch.zeros((capacity + 1, 6), dtype=torch.float64, device=device)
        if rank == src:
            k = min(capacity, len(strokes) - start)
            packed = np.zeros((capacity + 1, 6), dtype=np.float64)
            packed[0, 0], packed[0, 1] = k, len(strokes) - start - k       # this round, still to come
            packed[1:k + 1, :4] = strokes[start:start + k]
            packed[1:k + 1, 4] = layer_of[start:start + k]
            packed[1:k + 1, 5] = values[start:start + k]                   # uint32 bit patterns are exact in float64
            buf.copy_(torch.from_numpy(packed))
            start += k
        dist.broadcast(buf, src=src)
        out = buf.cpu().numpy()
        k, more = int(out[0, 0]), int(out[0, 1])
        outs.append(out[1:k + 1])
        if more <= 0:
            break
    out = np.concatenate(outs, axis=0)
    return (np.ascontiguousarray(out[:, :4]), out[:, 4].astype(np.int32), out[:, 5].astype(np.uint32))


def broadcast_batch(batch, src=0):
    """Device-to-device broadcast of a ``_native.StrokeBatch``'s packed record buffer (rank ``src`` has called
    ``batch.upload(..., fill=True)``; every rank's batch was created with the same ``capacity``).  One
    collective on the compute stream, no host read-back: receivers use the whole buffer (unused slots hold
    NaN strokes, which hit nothing), so the stroke path never waits for the host."""
    dist = _dist()
    _, ws = world()
    if ws > 1:
        dist.broadcast(batch.packed, src=src)
    return batch.use(batch._cap)


class AreaReducer:
    """Cross-rank sum of the per-layer areas (float64) and texel counts (int64) with ONE collective and no
    conversion kernels: every rank's 2L raw 8-byte slots are all-gathered (a few hundred bytes) and summed
    locally in rank order, so all ranks get bit-identical areas whatever algorithm the backend picks for an
    all-reduce.  ``slots``: int64 tensor of 2L elements, [0, L) holding the float64 bit patterns of the
    partial sums (the area kernel writes them through a float64 view), [L, 2L) the counts."""

    def __init__(self, layers, device):
        import torch
        self.L = int(layers)
        _, self.ws = world()
        self.gathered = torch.empty((self.ws, 2 * self.L), dtype=torch.int64, device=device) if self.ws > 1 else None

    def __call__(self, slots):
        if self.ws == 1:
            return slots
        import torch
        dist = _dist()
        if slots.is_cuda and dist.get_backend() != "nccl":
            # gloo (CPU tests, single-GPU rehearsal of the multi-rank path) gathers host tensors only
            host = [torch.empty(2 * self.L, dtype=torch.int64) for _ in range(self.ws)]
            dist.all_gather(host, slots.cpu())
            self.gathered.copy_(torch.stack(host))
        else:
            dist.all_gather_into_tensor(self.gathered.view(-1), slots.contiguous())
        L = self.L
        slots[:L].view(torch.float64).copy_(self.gathered[:, :L].view(torch.float64).sum(dim=0))
        slots[L:].copy_(self.gathered[:, L:].sum(dim=0))
        return slots


def agree(flag, device=None):
    """True iff ``flag`` is true on EVERY rank (one all-reduce; ranks reach it whatever happened locally)."""
    import torch
    dist = _dist()
    _, ws = world()
    if ws == 1:
        return bool(flag)
    t = torch.tensor([1 if flag else 0], dtype=torch.int64)
    if dist.get_backend() == "nccl":
        t = t.to(device if device is not None else torch.device("cuda", torch.cuda.current_device()))
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return int(t.item()) == 1


class PeerAreaReducer:
    """Fused compute + collective for the per-layer areas: no collective call at all.  Every rank owns a ring of
    result rows in an IPC-exported region; the area reduction kernel of every rank adds its per-block partials with
    system-scope atomics into the step's row of EVERY rank (NVLink peer memory), one thread then signals / awaits the
    arrival slots (``_native.layer_area_peers``).  ``reduce(step, area, masks, out)`` leaves the global sums and counts
    of all L layers in ``out`` (int64[2L], sums as float64 bit patterns) on every rank.

    Set-up (once): regions are allocated with cudaMalloc, the 64-byte IPC handles travel through the default process
    group (host side), every rank maps every other rank's region.  Rows are recycled NSLOTS steps later; a row is
    zeroed by its owner half a ring ahead, right after the wait of the current step -- at that point every rank has
    finished the current step (that is what the wait established) and none is further than one step ahead."""

    NSLOTS = 16

    def __init__(self, layers, device):
        import torch
        from . import _native
        dist = _dist()
        self.L = int(layers)
        self.rank, self.ws = world()
        self.device = device
        self.row_bytes = (2 * self.L + 2) * 8
        self.region = _native.PeerRegion(self.NSLOTS * self.row_bytes)
        handles = [None] * self.ws
        dist.all_gather_object(handles, (self.region.handle, int(torch.cuda.current_device())))
        # Mapping the peers can fail on ONE rank only (no peer atomics on some link, IPC not permitted); the ranks must
        # leave this constructor together, so the local failure is kept until all of them have voted.
        failure = None
        self.peers = [self.region]
        try:
            for _, peer_dev in handles:
                if not _native.lib().ml_peer_atomics_supported(int(peer_dev)):
                    raise RuntimeError("no native peer atomics between cuda:%d and cuda:%d" % (torch.cuda.current_device(), peer_dev))
            self.peers = [self.region if r == self.rank else _native.PeerRegion.open(handles[r][0], self.region.nbytes)
                          for r in range(self.ws)]
            self.own = self.region.tensor(torch.int64, device).view(self.NSLOTS, 2 * self.L + 2)
            # per slot: the addresses of every rank's arrival slot, as a device table
            self.arrive = torch.tensor([[p.ptr + s * self.row_bytes + 2 * self.L * 8 for p in self.peers] for s in range(self.NSLOTS)],
                                       dtype=torch.int64, device=device)
            self.status = torch.zeros(1, dtype=torch.int32, device=device)
        except Exception as exc:
            failure = exc
        # the vote is also the barrier: every region is mapped everywhere before anybody adds into one
        if not agree(failure is None, device):
            self.close()
            raise RuntimeError("peer regions could not be mapped on every rank (%s)" % (failure or "another rank failed"))

    def self_test(self):
        """One trial reduction with known contributions (rank r adds r + 1 for each of 4096 texels into every layer):
        True iff this rank's row then holds the expected global sums and counts and the wait did not time out.  Uses
        the last slot of the ring and leaves it zeroed (it is recycled again long before its first real use)."""
        import torch
        from . import _native
        n = 4096
        area = torch.full((1, n), float(self.rank + 1), dtype=torch.float32, device=self.device)
        mask = torch.ones((1, n), dtype=torch.uint8, device=self.device)
        s = self.NSLOTS - 1
        rows = [p.ptr + s * self.row_bytes for p in self.peers]
        _native.layer_area_peers(area, [mask] * self.L, rows, self.rank, self.arrive[s], self.status)
        got = self.own[s, :2 * self.L].clone()
        self.own[s].zero_()
        got = got.cpu()
        want_sum = float(n * sum(r + 1 for r in range(self.ws)))
        ok = (not int(self.status.item())
              and bool((got[:self.L].view(torch.float64) == want_sum).all())
              and bool((got[self.L:] == n * self.ws).all()))
        return ok

    def reduce(self, step, area, masks, out):
        from . import _native
        s = step % self.NSLOTS
        ahead = (step + self.NSLOTS // 2) % self.NSLOTS
        rows = [p.ptr + s * self.row_bytes for p in self.peers]
        _native.layer_area_peers(area, masks, rows, self.rank, self.arrive[s], self.status,
                                 recycle_row=self.region.ptr + ahead * self.row_bytes)
        out.copy_(self.own[s, :2 * self.L])
        return out

    def check(self):
        if int(self.status.item()):
            raise RuntimeError("peer area reduction timed out waiting for another rank")

    def close(self):
        for p in self.peers:
            if p is not self.region:
                p.close()
        self.peers = [self.region]
        self.region.close()


def allreduce_areas(sums, counts=None):
    """Sum per-layer partial areas (float64 tensor) and counts (int64 tensor) over all ranks, in
    place.  One collective: counts ride along as exact float64 (< 2^53 texels).  (Convenience form;
    the per-step path uses ``AreaReducer``, which needs no packing kernels.)"""
    import torch
    dist = _dist()
    _, ws = world()
    if ws == 1:
        return sums, counts
    if counts is None:
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
        return sums, None
    packed = torch.cat([sums, counts.to(torch.float64)])
    dist.all_reduce(packed, op=dist.ReduceOp.SUM)
    n = sums.numel()
    sums.copy_(packed[:n])
    counts.copy_(packed[n:].round().to(torch.int64))
    return sums, counts


def allreduce_counts(counts):
    """Sum int64 edit counters over ranks, in place."""
    dist = _dist()
    _, ws = world()
    if ws > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM)
    return counts


def halo_bounds(row0, rows, height, radius):
    """Rows a rank needs for a radius-``radius`` stencil: (in_row0, in_rows) clipped to the atlas."""
    lo = max(0, row0 - radius)
    hi = min(height, row0 + rows + radius)
    return lo, hi - lo


def exchange_halo(plane, row0, height, radius, parts=False):
    """Return the rank's slab of a byte plane extended by up to ``radius`` rows from each
    neighbour, plus the global row index of its first row.  Neighbour rows travel point-to-point
    (isend/irecv); interior-only when world_size == 1.  ``parts=True`` returns the received rows
    alone, ``(rows_from_above_or_None, rows_from_below_or_None)``, without building the extended
    plane (per-stroke path: the slab is 268 MB, the halo 16 KB)."""
    import torch
    dist = _dist()
    rank, ws = world()
    rows = plane.shape[0]
    if ws == 1 or radius <= 0:
        return (None, None) if parts else (plane, row0)
    up_n = min(radius, row0)                                   # rows needed from rank-1 (above = lower rows)
    dn_n = min(radius, height - (row0 + rows))
    # all four transfers go into ONE batch (ncclGroupStart/End under NCCL): posting them one by one
    # would deadlock, every rank's first operation being a receive.  NCCL moves device rows directly;
    # any other backend (gloo: CPU tests, single-GPU rehearsal of the multi-rank path) gets the few
    # halo rows staged through host memory, because its point-to-point ops take host tensors only.
    xdev = plane.device if (dist.get_backend() == "nccl" or not plane.is_cuda) else torch.device("cpu")
    ops, up, dn = [], None, None
    if rank > 0:
        up = torch.empty((up_n,) + tuple(plane.shape[1:]), dtype=plane.dtype, device=xdev)
        ops.append(dist.P2POp(dist.irecv, up, rank - 1))
        ops.append(dist.P2POp(dist.isend, plane[:min(radius, rows)].contiguous().to(xdev), rank - 1))
    if rank < ws - 1:
        dn = torch.empty((dn_n,) + tuple(plane.shape[1:]), dtype=plane.dtype, device=xdev)
        ops.append(dist.P2POp(dist.irecv, dn, rank + 1))
        ops.append(dist.P2POp(dist.isend, plane[max(0, rows - radius):].contiguous().to(xdev), rank + 1))
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    up = up.to(plane.device) if up is not None else None
    dn = dn.to(plane.device) if dn is not None else None
    if parts:
        return up, dn
    pieces = [p for p in (up, plane, dn) if p is not None]
    return torch.cat(pieces, dim=0), row0 - (up.shape[0] if up is not None else 0)


def exchange_halo_into(buf, margin, rows, row0, height, radius):
    """Per-stroke form of ``exchange_halo``: ``buf`` is a rank's byte plane allocated with ``margin`` spare rows above
    and below its ``rows`` slab rows (the slab is ``buf[margin:margin + rows]``); the neighbours' ``radius`` border rows
    are received STRAIGHT INTO those spare rows (no concatenation, no allocation: round 1 built two ``torch.cat``
    windows per stroke).  Returns ``(up_n, dn_n)``, the rows now valid above / below the slab."""
    import torch
    dist = _dist()
    rank, ws = world()
    if ws == 1 or radius <= 0:
        return 0, 0
    if radius > margin:
        raise ValueError("halo radius exceeds the plane's spare rows")
    up_n = min(radius, row0)
    dn_n = min(radius, height - (row0 + rows))
    slab = buf[margin:margin + rows]
    direct = dist.get_backend() == "nccl" or not buf.is_cuda
    ops, stage_up, stage_dn = [], None, None
    if rank > 0:
        dst = buf[margin - up_n:margin]
        stage_up = dst if direct else torch.empty(dst.shape, dtype=dst.dtype)
        ops.append(dist.P2POp(dist.irecv, stage_up, rank - 1))
        src = slab[:min(radius, rows)]
        ops.append(dist.P2POp(dist.isend, src if direct else src.cpu(), rank - 1))
    if rank < ws - 1:
        dst = buf[margin + rows:margin + rows + dn_n]
        stage_dn = dst if direct else torch.empty(dst.shape, dtype=dst.dtype)
        ops.append(dist.P2POp(dist.irecv, stage_dn, rank + 1))
        src = slab[max(0, rows - radius):]
        ops.append(dist.P2POp(dist.isend, src if direct else src.cpu(), rank + 1))
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    if not direct:                      # gloo with device planes (single-GPU rehearsal): staged through the host
        if stage_up is not None:
            buf[margin - up_n:margin].copy_(stage_up)
        if stage_dn is not None:
            buf[margin + rows:margin + rows + dn_n].copy_(stage_dn)
    return (up_n if rank > 0 else 0), (dn_n if rank < ws - 1 else 0)
