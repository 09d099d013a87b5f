"""Multi-GPU orchestration of the ID: one process per GPU, torch.distributed
(NCCL over NVLink/NVSwitch on the B200 box; gloo for the CPU tests).

Perspectives are independent, so the path shards across ranks with exactly two kinds of
exchange, both real data movement of the method:

* map replication -- the packed 2-bit store (4 MiB at 256^3, 32 MiB at 512^3) is
  broadcast once from the rank that built it, and each cycle's map deltas (KB-scale)
  are broadcast so every replica applies the same update (the single-writer rule,
  S:97-98, holds per replica by stream order);
* depth frames (row f3) -- the sensor rank broadcasts each frame's points and every
  replica integrates it (deterministic, so the maps stay identical);
* the IG point cloud -- each rank computes a strided slice of the perspective set
  (perspective j -> rank j mod G, so cheap in-object and expensive open-space
  perspectives spread evenly), and one all-gather assembles the cloud in input order on
  every rank, where the IDW query runs;
* the ray split (fewer perspectives than GPUs, e.g. one perspective at full resolution):
  every rank walks its share of each perspective's rays and one all-reduce sums the
  integer totals before the finalize.

The collectives run on torch's current stream, so the library ctx must use that stream
(nbt.Ctx(device, torch.cuda.current_stream().cuda_stream)) for stream order to hold.
Integer per-state totals make the result bit-identical to a single-GPU run (the g_P of a
perspective depends only on its own totals).  The arithmetic stays in libnbt; this module
only moves tensors.
"""
from __future__ import annotations

import os

import numpy as np


def env_rank_world():
    """(rank, world, local_rank) from the torchrun environment (1 process if absent)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def init_process_group(backend="nccl"):
    """Join the torchrun job.  NBT_DIST_BACKEND=gloo overrides the backend and maps every
    rank onto the visible GPUs round-robin: a functional check of the multi-rank path on a
    one-GPU box (collectives through the host, so no rank's kernel waits on another's);
    returns local = the CUDA device to use."""
    import torch.distributed as dist
    rank, world, local = env_rank_world()
    override = os.environ.get("NBT_DIST_BACKEND")
    if override:
        backend = override
        if backend != "nccl":
            import torch
            if torch.cuda.is_available():
                local = local % torch.cuda.device_count()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


# ------------------------------------------------------------------ shard logic

def shard_count(n: int, rank: int, world: int) -> int:
    """Number of perspectives j < n with j mod world == rank."""
    return max(0, (n - rank + world - 1) // world) if rank < n else 0


def rows_per_rank(n: int, world: int) -> int:
    return (n + world - 1) // world


def unstride(gathered, n: int, world: int):
    """gathered: (world, R, ...) with rank r's rows r, r+W, r+2W, ... padded to R.
    Returns the (n, ...) array in the original perspective order."""
    R = gathered.shape[1]
    tail = tuple(gathered.shape[2:])
    if hasattr(gathered, "transpose") and not isinstance(gathered, np.ndarray):
        flat = gathered.transpose(0, 1).reshape((world * R,) + tail)
    else:
        flat = np.swapaxes(gathered, 0, 1).reshape((world * R,) + tail)
    return flat[:n]


def pad_rows(t, rows: int):
    """Pad a (k, ...) tensor to (rows, ...) with NaN / zeros (dropped after the gather)."""
    import torch
    k = t.shape[0]
    if k == rows:
        return t.contiguous()
    fill = float("nan") if t.dtype.is_floating_point else 0
    out = torch.full((rows,) + tuple(t.shape[1:]), fill, dtype=t.dtype, device=t.device)
    out[:k] = t
    return out


# ------------------------------------------------------------------ collectives

class _CudaBytes:
    """__cuda_array_interface__ view of a raw device allocation (the packed map)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3}


def map_tensor(m):
    """A uint8 CUDA tensor aliasing the map's packed store (no copy)."""
    import torch
    ptr, nbytes = m.device_buffer()
    return torch.as_tensor(_CudaBytes(ptr, nbytes), device=torch.device("cuda", m.ctx.device))


def replicate_map(m, src: int = 0, group=None):
    """Broadcast the packed store of `src`'s map into every rank's map (same desc)."""
    import torch.distributed as dist
    m.ctx.sync()
    dist.broadcast(map_tensor(m), src=src, group=group)


def broadcast_deltas(ijk, codes, src: int = 0, group=None):
    """Broadcast one cycle's map deltas (device tensors of equal shape on every rank)."""
    import torch.distributed as dist
    dist.broadcast(ijk, src=src, group=group)
    dist.broadcast(codes, src=src, group=group)


def broadcast_frame(points, sensor, src: int = 0, device=None, group=None):
    """Broadcast one depth frame (row f3) from the sensor rank: (sensor float64[3], points
    float64 [n, 3] tensor on `device`) on every rank.  Other ranks pass points=None.  Every
    replica then integrates the same frame; the integration is deterministic (per-cloud set
    update, Q35), so the replicated maps stay bit-identical without a delta exchange."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    head = torch.zeros(4, dtype=torch.float64, device=device)
    if rank == src:
        pts = torch.as_tensor(points, dtype=torch.float64).reshape(-1, 3).to(device)
        head[0] = float(pts.shape[0])
        head[1:] = torch.as_tensor(np.asarray(sensor, dtype=np.float64), device=device)
    dist.broadcast(head, src=src, group=group)
    n = int(head[0].item())
    if rank != src:
        pts = torch.empty((n, 3), dtype=torch.float64, device=device)
    if n:
        dist.broadcast(pts, src=src, group=group)
    return head[1:].cpu().numpy(), pts.contiguous()


def integrate_replicated(occ, m, points, sensor, params=None, src: int = 0, group=None):
    """Row f3 on every replica: broadcast the frame from `src`, integrate it locally."""
    import torch
    dev = torch.device("cuda", occ.ctx.device)
    sensor, pts = broadcast_frame(points, sensor, src=src, device=dev, group=group)
    occ.integrate(sensor, pts, map=m, params=params)


def all_gather_rows(local, n_total: int, world: int, strided: bool = True, group=None):
    """All-gather per-rank row blocks into the full (n_total, ...) array on every rank.
    strided=True: rank r holds rows r, r+W, ... (shard_count rows); False: contiguous
    equal blocks (weak scaling: rank r holds rows r*k .. r*k + k-1)."""
    import torch
    import torch.distributed as dist
    R = rows_per_rank(n_total, world) if strided else local.shape[0]
    loc = pad_rows(local, R)
    out = torch.empty((world * R,) + tuple(loc.shape[1:]), dtype=loc.dtype, device=loc.device)
    dist.all_gather_into_tensor(out, loc, group=group)
    if not strided:
        return out[:n_total]
    return unstride(out.view((world, R) + tuple(loc.shape[1:])), n_total, world)


def gather_cloud(local_xyz, local_gain, local_counts, n_total: int, world: int, strided: bool = True,
                 out=None, group=None):
    """One all-gather of this rank's IG-cloud rows packed as 64-byte rows (xyz 3 x f64, g_P f64,
    counts 4 x u64 bit-cast), un-strided on every rank.  out = (xyz, gain, counts) tensors of
    n_total rows to fill (else new ones); returns them."""
    import torch
    k = local_gain.shape[0]
    rows = torch.empty((k, 8), dtype=torch.float64, device=local_gain.device)
    rows[:, :3] = local_xyz
    rows[:, 3] = local_gain
    rows[:, 4:] = local_counts.view(torch.float64)
    full = all_gather_rows(rows, n_total, world, strided=strided, group=group)
    if out is None:
        out = (torch.empty((n_total, 3), dtype=torch.float64, device=rows.device),
               torch.empty(n_total, dtype=torch.float64, device=rows.device),
               torch.empty((n_total, 4), dtype=torch.int64, device=rows.device))
    out[0].copy_(full[:, :3])
    out[1].copy_(full[:, 3])
    out[2].copy_(full[:, 4:].contiguous().view(torch.int64))
    return out


def id_compute_sharded(nbt, ctx, m, poi, persp_dev, cam, range_, rank: int, world: int, group=None):
    """The whole ID of `persp_dev` (n x 3 CUDA tensor, identical on every rank), sharded
    j -> rank j mod world, gathered in input order on every rank: (xyz, gain, counts)."""
    import torch
    n = persp_dev.shape[0]
    k = shard_count(n, rank, world)
    dev = persp_dev.device
    local = nbt.IgCloud(torch.empty((k, 3), dtype=torch.float64, device=dev),
                        torch.empty(k, dtype=torch.float64, device=dev),
                        torch.empty((k, 4), dtype=torch.int64, device=dev))
    if k:
        nbt.id_compute(ctx, m, poi, persp_dev, cam, range_, out=local, first=rank, stride=world)
    if world == 1:
        return local.xyz, local.gain, local.counts
    return gather_cloud(local.xyz, local.gain, local.counts, n, world, group=group)


def id_compute_ray_split(nbt, ctx, m, poi, persp_dev, cam, range_, rank: int, world: int, group=None):
    """The whole ID of `persp_dev` (n x 3 CUDA tensor, identical on every rank) with the RAYS
    of every perspective sharded over the ranks (SURVEY 8(e) ray split, for N_P < G): each
    rank walks its 32-ray units, the integer totals are summed by one all-reduce (exact), and
    every rank finalizes the same cloud, bit-identical to one GPU: (xyz, gain, counts)."""
    import torch
    import torch.distributed as dist
    totals = nbt.id_compute_rays(ctx, m, poi, persp_dev, cam, range_, rank, world)
    if world > 1:
        dist.all_reduce(totals, op=dist.ReduceOp.SUM, group=group)
    n = persp_dev.shape[0]
    dev = persp_dev.device
    cloud = nbt.IgCloud(torch.empty((n, 3), dtype=torch.float64, device=dev),
                        torch.empty(n, dtype=torch.float64, device=dev),
                        torch.empty((n, 4), dtype=torch.int64, device=dev))
    nbt.id_finalize(ctx, m, poi, persp_dev, cam, range_, totals, out=cloud)
    return cloud.xyz, cloud.gain, cloud.counts


class PeerUnavailable(RuntimeError):
    """Some rank could not map a peer's buffer (raised on every rank alike)."""


def make_peer_gather(nbt, ctx, rows: int, rank: int, world: int, group=None, n_buffers: int = 2):
    """A PeerGather, or None (on every rank) when peer mapping is unavailable: the caller then
    uses the NCCL all-gather (id_compute_sharded / all_gather_rows) instead."""
    try:
        return PeerGather(nbt, ctx, rows, rank, world, group=group, n_buffers=n_buffers)
    except PeerUnavailable:
        return None


class PeerGather:
    """The IG-cloud all-gather fused into the finalize over peer memory (nbt_gather_*): two
    library-owned row buffers per rank (alternated between cycles, so a rank never rewrites a
    buffer a peer may still read), their CUDA IPC handles exchanged once through the process
    group, every peer's buffers mapped.  Each cycle, every rank's finalize stores its rows
    into all ranks' current buffers; a stream sync plus a process barrier then orders the
    readers after every rank's stores (no kernel waits on another rank's kernel)."""

    def __init__(self, nbt, ctx, rows: int, rank: int, world: int, group=None, n_buffers: int = 2):
        import torch.distributed as dist
        self.nbt, self.ctx, self.rows, self.rank, self.world, self.group = nbt, ctx, rows, rank, world, group
        self.bufs = [nbt.Gather(ctx, rows, world, rank) for _ in range(n_buffers)]
        mine = [g.export() for g in self.bufs]
        everyone = [None] * world
        dist.all_gather_object(everyone, mine, group=group)
        err = None
        try:
            for g_idx, g in enumerate(self.bufs):
                for r in range(world):
                    if r != rank:
                        g.attach(r, everyone[r][g_idx])
        except nbt.NbtError as e:      # e.g. CUDA IPC unavailable between these processes
            err = str(e)
        # every rank learns whether every rank could map every peer
        errs = [None] * world
        dist.all_gather_object(errs, err, group=group)
        bad = [f"rank {r}: {x}" for r, x in enumerate(errs) if x]
        if bad:
            self.close()
            raise PeerUnavailable("; ".join(bad))
        self.cycle = 0

    def id_compute(self, m, poi, persp_dev, cam, range_):
        """The whole ID of `persp_dev` (identical on every rank), perspective j computed by rank
        j mod world and stored into every rank's buffer: returns this rank's (xyz, gain, counts)
        CUDA tensors viewing the current buffer (valid until the buffer is reused two cycles on)."""
        import torch.distributed as dist
        g = self.bufs[self.cycle % len(self.bufs)]
        self.cycle += 1
        g.compute(m, poi, persp_dev, cam, range_)
        self.order_readers()
        c = g.cloud()
        return c.xyz, c.gain, c.counts

    def order_readers(self):
        """Order every later read of this rank (in its stream) after all ranks' stores: a
        word-sized all-reduce on the stream under NCCL (no host synchronisation); gloo works
        on the host, so there the stream is drained first."""
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return
        if dist.get_backend(self.group) != "nccl":
            self.ctx.sync()
        if not hasattr(self, "_token"):
            self._token = torch.zeros(1, dtype=torch.int64, device=torch.device("cuda", self.ctx.device))
        dist.all_reduce(self._token, group=self.group)

    def ray_split(self, m, poi, persp_dev, cam, range_):
        """The ID with the RAYS of every perspective sharded over the ranks and the totals'
        all-reduce fused into the walk (remote atomics into every rank's buffer): returns the
        same (xyz, gain, counts) on every rank, bit-identical to one GPU."""
        import torch
        g = self.bufs[self.cycle % len(self.bufs)]     # never the buffer an earlier result views
        self.cycle += 1
        n = persp_dev.shape[0]
        g.zero()
        self.order_readers()                 # every rank's clear before any rank's adds
        g.compute_rays(m, poi, persp_dev, cam, range_)
        self.order_readers()                 # every rank's adds before the finalize
        dev = persp_dev.device
        cloud = self.nbt.IgCloud(torch.empty((n, 3), dtype=torch.float64, device=dev),
                                 torch.empty(n, dtype=torch.float64, device=dev),
                                 torch.empty((n, 4), dtype=torch.int64, device=dev))
        self.nbt.id_finalize(self.ctx, m, poi, persp_dev, cam, range_, g.totals(n), out=cloud)
        return cloud.xyz, cloud.gain, cloud.counts

    def close(self):
        for g in self.bufs:
            g.close()
