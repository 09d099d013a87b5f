import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_22588_b200 as nbt
from nbt_inputs import CONFIGS, FOV_H, FOV_V
cfg = CONFIGS["B"]
dev = torch.device("cuda", 0); st = torch.cuda.Stream(dev); torch.cuda.set_stream(st)
ctx = nbt.Ctx(0, st.cuda_stream)
m = nbt.Map(ctx, nbt.map_desc(cfg.n, cfg.n, cfg.n, cfg.voxel_size)); m.upload(cfg.map_codes())
cam = nbt.camera_from_grid_scaling(FOV_H, FOV_V, 3.86, cfg.voxel_size, 5.0)
ctx.set_profiling(True)
for (n, seed) in [(100, 107), (200, 207), (100, 207), (200, 107), (1000, 1007), (50, 107), (25, 107)]:
    P = nbt.sample_perspectives(ctx, cfg.poi, cfg.persp_radius, n, seed, 0)
    if n == 100 and seed == 207:
        P = nbt.sample_perspectives(ctx, cfg.poi, cfg.persp_radius, 200, 207, 0)[:100].copy()
    if n == 200 and seed == 107:
        P = np.concatenate([nbt.sample_perspectives(ctx, cfg.poi, cfg.persp_radius, 100, 107, 0)] * 2)
    out = nbt.empty_cloud(n, device=dev)
    Pd = torch.from_numpy(P).to(dev)
    for _ in range(3): nbt.id_compute(ctx, m, cfg.poi, Pd, cam, 3.86, out=out)
    ctx.sync(); ctx.profile_read(0, reset=True)
    for _ in range(10): nbt.id_compute(ctx, m, cfg.poi, Pd, cam, 3.86, out=out)
    ms, k = ctx.profile_read(0, reset=True)
    c = out.counts.cpu().numpy()
    print(json.dumps({"n": n, "seed": seed, "trace_ms": ms / k, "lookups": float(c[:, 3].sum()),
                      "max_persp_lookups": float(c[:, 3].max()), "mean_persp_lookups": float(c[:, 3].mean())}))
