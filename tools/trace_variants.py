"""Time the trace kernel on config workloads (device-resident inputs, CUDA events around
each k_id_trace launch).  Experiment knobs: --layout linear|morton and --bits 2|8 (the map
descriptor), --opt NAME=VALUE (ctx options, e.g. --opt TRACE_REFILL_MIN=8); --prob uses the
8-bit per-voxel-probability store (f1); NBT_LIB=<path> loads a variant library build.

    python tools/trace_variants.py B "C'" D [--prob] [--layout morton] [--bits 8] [--opt TRACE_CARVEOUT=50]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_2503_22588_b200 as nbt
from nbt_inputs import CONFIGS, FOV_H, FOV_V


def run(cfg_name, reps=5, prob=False, layout="linear", bits=2, opts=(), persp=None, stride=1, offset=0,
        ray_world=1, ray_rank=0):
    cfg = CONFIGS[cfg_name]
    n_use = persp if persp else cfg.n_persp
    dev = torch.device("cuda", 0)
    s = torch.cuda.Stream(dev)
    torch.cuda.set_stream(s)
    ctx = nbt.Ctx(0, s.cuda_stream)
    for name, value in opts:
        ctx.set_option(getattr(nbt, "OPT_" + name), value)
    m = nbt.Map(ctx, nbt.map_desc(cfg.n, cfg.n, cfg.n, cfg.voxel_size, layout=layout, state_bits=bits), prob=prob)
    codes = cfg.map_codes()
    if prob:      # per-voxel probabilities: Free P in [0.12, 0.5), Occupied in [0.5, 0.97]
        rng = np.random.default_rng(0)
        u = rng.random(codes.shape, dtype=np.float32)
        p = np.where(codes == 1, 0.12 + 0.38 * u, 0.5 + 0.47 * u).astype(np.float32)
        m.upload_prob(p, (codes != 0).astype(np.uint8))
    else:
        m.upload(codes)
    cam = nbt.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
    persp_all = torch.empty((cfg.n_persp, 3), dtype=torch.float64, device=dev)
    nbt.sample_perspectives(ctx, cfg.poi, cfg.persp_radius, cfg.n_persp, cfg.persp_seed, cfg.persp_mode,
                            out=persp_all)
    # --persp N --stride S: N perspectives j = 0, S, 2S, ... (one rank's strided shard of D at S ranks)
    persp = persp_all[offset::stride][:n_use].contiguous()
    out = nbt.empty_cloud(persp.shape[0], device=dev)
    if ray_world > 1:
        # --ray-world W --ray-rank R: ray shard R of W of every perspective (the ray split)
        def one():
            return nbt.id_compute_rays(ctx, m, cfg.poi, persp, cam, cfg.range_, ray_rank, ray_world)
    else:
        def one():
            return nbt.id_compute(ctx, m, cfg.poi, persp, cam, cfg.range_, out=out)
    one()
    ctx.sync()
    ctx.set_profiling(True)
    ctx.profile_read(nbt.KERNEL_TRACE, reset=True)
    for _ in range(reps):
        res = one()
    ms, n = ctx.profile_read(nbt.KERNEL_TRACE, reset=True)
    counts = res.cpu().numpy()[:, :4] if ray_world > 1 else out.counts.cpu().numpy()
    lookups = float(counts[:, 3].sum())
    ms /= n
    rays = cfg.rays_per_id // cfg.n_persp * persp.shape[0] // ray_world
    return {"config": cfg_name, "store": "8-bit prob" if prob else f"{bits}-bit {layout}", "trace_ms": ms,
            "persp": int(persp.shape[0]), "rays_per_s": rays / (ms / 1e3), "lookups_per_s": lookups / (ms / 1e3),
            "lookups": lookups, "checksum": int(counts.sum())}


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["B"])
    ap.add_argument("--prob", action="store_true")
    ap.add_argument("--layout", default="linear")
    ap.add_argument("--bits", type=int, default=2)
    ap.add_argument("--opt", action="append", default=[])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--persp", type=int, default=None, help="use N of the config's perspectives")
    ap.add_argument("--stride", type=int, default=1, help="... taking every S-th (a strided rank shard)")
    ap.add_argument("--offset", type=int, default=0, help="... starting at this one (the rank)")
    ap.add_argument("--ray-world", type=int, default=1, help="ray split: shards of every perspective's rays")
    ap.add_argument("--ray-rank", type=int, default=0, help="... this shard")
    a = ap.parse_args()
    opts = [(o.split("=")[0], int(o.split("=")[1])) for o in a.opt]
    for name in a.configs:
        print(json.dumps(run(name, reps=a.reps, prob=a.prob, layout=a.layout, bits=a.bits, opts=opts,
                             persp=a.persp, stride=a.stride, offset=a.offset, ray_world=a.ray_world,
                             ray_rank=a.ray_rank)), flush=True)
