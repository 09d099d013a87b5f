"""Multi-rank functional check of the sharded path, launched by torchrun:

    torchrun --nproc-per-node G tools/multirank_check.py
    NBT_DIST_BACKEND=gloo torchrun --nproc-per-node 2 tools/multirank_check.py   # one-GPU box

Every rank holds a replica of the map (NCCL / gloo broadcast of the packed store), applies
the same broadcast deltas, computes its strided shard of an ID and all-gathers the IG cloud,
walks its ray shard of a few perspectives and all-reduces the integer totals (ray split),
gathers the cloud through peer memory with the finalize-fused all-gather (nbt_gather_*),
and integrates the same broadcast depth frame.  Checks, across ranks: identical map and
occupancy replicas (digests), and a gathered cloud bit-identical to the unsharded ID that
rank 0 computes with the same library.  Uses only libnbt (no oracle).  Prints
"MULTIRANK OK <world>" on rank 0 and exits 0, else raises.
"""
import hashlib
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_22588_b200 as nbt  # noqa: E402
from paper_2503_22588_b200 import dist as ndist  # noqa: E402
from nbt_inputs import CLOUD_CONFIGS, CONFIGS, FOV_H, FOV_V, cycle_deltas  # noqa: E402


def digest(a) -> int:
    b = np.ascontiguousarray(a).tobytes()
    return int.from_bytes(hashlib.sha256(b).digest()[:7], "little")


def same_everywhere(value: int, world: int, dev) -> bool:
    t = torch.tensor([value], dtype=torch.int64, device=dev)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return all(int(o.item()) == value for o in out)


def main():
    rank, world, local = ndist.init_process_group(os.environ.get("NBT_DIST_BACKEND", "nccl"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = nbt.Ctx(local, stream.cuda_stream)
    cfg = CONFIGS["A"]
    desc = nbt.map_desc(cfg.n, cfg.n, cfg.n, cfg.voxel_size)
    m = nbt.Map(ctx, desc)
    codes = cfg.map_codes()
    if rank == 0:
        m.upload(codes)
    ndist.replicate_map(m, src=0)
    ctx.sync()
    assert same_everywhere(digest(m.download()), world, dev), "map replicas differ after broadcast"
    assert rank != 0 or np.array_equal(m.download(), codes)

    # one cycle of deltas from the sensor rank
    ijk, vals = cycle_deltas(cfg.n, (cfg.n // 2,) * 3, 3, codes, seed=1)
    n_d = torch.tensor([len(vals)], dtype=torch.int64, device=dev)
    dist.broadcast(n_d, src=0)
    d_ijk = torch.from_numpy(ijk).to(dev) if rank == 0 else torch.zeros((int(n_d.item()), 3), dtype=torch.int32,
                                                                         device=dev)
    d_val = torch.from_numpy(vals).to(dev) if rank == 0 else torch.zeros(int(n_d.item()), dtype=torch.uint8,
                                                                         device=dev)
    ndist.broadcast_deltas(d_ijk, d_val, src=0)
    m.update(d_ijk, d_val)
    ctx.sync()
    assert same_everywhere(digest(m.download()), world, dev), "map replicas differ after the deltas"

    # sharded ID gathered in input order == the unsharded ID
    n_p = 37                                     # not a multiple of the world size
    persp = torch.empty((n_p, 3), dtype=torch.float64, device=dev)
    nbt.sample_perspectives(ctx, cfg.poi, cfg.persp_radius, n_p, 11, cfg.persp_mode, out=persp)
    cam = nbt.camera_from_fov(FOV_H, FOV_V, 24, 18)
    xyz, gain, counts = ndist.id_compute_sharded(nbt, ctx, m, cfg.poi, persp, cam, cfg.range_, rank, world)
    torch.cuda.synchronize()
    full = nbt.id_compute(ctx, m, cfg.poi, persp, cam, cfg.range_)
    ctx.sync()
    assert torch.equal(xyz, persp), "gathered perspectives out of order"
    assert np.array_equal(gain.cpu().numpy(), np.asarray(full.gain)), "sharded g_P differ"
    assert np.array_equal(counts.cpu().numpy().astype(np.uint64), np.asarray(full.counts).astype(np.uint64))

    # the all-gather fused into the finalize over peer memory (CUDA IPC; plain device stores
    # when the ranks share one GPU): every rank's buffer holds the unsharded ID, two cycles so
    # both alternating buffers are used
    pg = ndist.PeerGather(nbt, ctx, n_p, rank, world)
    for _ in range(2):
        xyz_p, gain_p, counts_p = pg.id_compute(m, cfg.poi, persp, cam, cfg.range_)
        assert torch.equal(xyz_p, persp), "peer gather: perspectives out of order"
        assert np.array_equal(gain_p.cpu().numpy(), np.asarray(full.gain)), "peer gather: g_P differ"
        assert np.array_equal(counts_p.cpu().numpy().astype(np.uint64), np.asarray(full.counts).astype(np.uint64))
        dist.barrier()
    pg.close()
    # weak-scaling form: each rank's own perspectives into rows rank*k .. rank*k + k-1, equal
    # to the collective all-gather of the ranks' own IDs
    k_own = 9
    own = torch.empty((k_own, 3), dtype=torch.float64, device=dev)
    nbt.sample_perspectives(ctx, cfg.poi, cfg.persp_radius, k_own, 100 + rank, cfg.persp_mode, out=own)
    mine = nbt.id_compute(ctx, m, cfg.poi, own, cam, cfg.range_, out=nbt.empty_cloud(k_own, device=dev))
    ctx.sync()
    want_g = ndist.all_gather_rows(mine.gain, k_own * world, world, strided=False)
    want_c = ndist.all_gather_rows(mine.counts, k_own * world, world, strided=False)
    pw = ndist.PeerGather(nbt, ctx, k_own * world, rank, world, n_buffers=1)
    pw.bufs[0].compute(m, cfg.poi, own, cam, cfg.range_, first=0, stride=1, row0=rank * k_own)
    ctx.sync()
    dist.barrier()
    got = pw.bufs[0].cloud()
    assert torch.equal(got.gain, want_g) and torch.equal(got.counts, want_c), "peer gather (weak form) differs"
    dist.barrier()
    pw.close()

    # the same ray split with the all-reduce fused into the walk: count flushes add straight
    # into every rank's buffer through the peer mappings
    pr = ndist.PeerGather(nbt, ctx, 16, rank, world, n_buffers=1)
    for _ in range(2):
        few2 = persp[:max(1, world - 1)].contiguous()
        xyz_f, gain_f, counts_f = pr.ray_split(m, cfg.poi, few2, cam, cfg.range_)
        ctx.sync()
        k2 = few2.shape[0]
        assert np.array_equal(gain_f.cpu().numpy(), np.asarray(full.gain)[:k2]), "fused ray split: g_P differ"
        assert np.array_equal(counts_f.cpu().numpy().astype(np.uint64), np.asarray(full.counts)[:k2].astype(np.uint64))
    dist.barrier()
    pr.close()

    # ray split (fewer perspectives than ranks): every rank walks its ray units of the same
    # perspectives, one all-reduce of the integer totals, the same cloud as the unsharded ID
    few = persp[:max(1, world - 1)].contiguous()
    xyz_r, gain_r, counts_r = ndist.id_compute_ray_split(nbt, ctx, m, cfg.poi, few, cam, cfg.range_, rank, world)
    ctx.sync()
    k = few.shape[0]
    assert torch.equal(xyz_r, few), "ray split: perspectives differ"
    assert np.array_equal(gain_r.cpu().numpy(), np.asarray(full.gain)[:k]), "ray split: g_P differ"
    assert np.array_equal(counts_r.cpu().numpy().astype(np.uint64), np.asarray(full.counts)[:k].astype(np.uint64))

    # sharded IDW queries over the gathered cloud == all queries on one rank
    buf = nbt.IdBuffer(ctx, 4, n_p)
    for _ in range(3):
        buf.push(nbt.IgCloud(xyz.contiguous(), gain.contiguous(), None), n_p)
    qs = torch.from_numpy(cfg.poi + np.random.default_rng(5).normal(0, 3.0, (101, 3))).to(dev)
    rows = (101 + world - 1) // world
    lo, hi = min(101, rank * rows), min(101, rank * rows + rows)
    mine = torch.zeros(rows, dtype=torch.float64, device=dev)
    if hi > lo:
        buf.query(qs[lo:hi], out=mine[:hi - lo])
    gathered = ndist.all_gather_rows(mine, 101, world, strided=False)
    full_q = torch.empty(101, dtype=torch.float64, device=dev)
    buf.query(qs, out=full_q)
    ctx.sync()
    assert torch.equal(gathered, full_q), "sharded IDW queries differ"

    # f3: the sensor rank's frame, integrated by every replica
    cf = CLOUD_CONFIGS["F0"]
    fdesc = nbt.map_desc(cf.n, cf.n, cf.n, cf.voxel_size)
    occ = nbt.OccMap(ctx, fdesc)
    fm = nbt.Map(ctx, fdesc)
    prm = nbt.integrate_params(cf.voxel_size, leaf=cf.leaf, max_range=cf.max_range)
    for k in range(2):
        pts = cf.cloud(k) if rank == 0 else None
        ndist.integrate_replicated(occ, fm, pts, cf.sensor(k) if rank == 0 else None, params=prm, src=0)
    ctx.sync()
    L = occ.download()
    assert same_everywhere(digest(np.nan_to_num(L, nan=-7.0)), world, dev), "occupancy replicas differ"
    assert same_everywhere(digest(fm.download()), world, dev), "integrated map replicas differ"
    assert occ.stats()[1] > 0

    dist.barrier()
    if rank == 0:
        print(f"MULTIRANK OK {world}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
