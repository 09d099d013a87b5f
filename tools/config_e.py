"""Config E: the receding-horizon loop.  200 MHP cycles; each cycle applies
that cycle's map deltas, samples 512 perspectives around a moving PoI, recomputes the ID,
pushes it into the N_B = 10 buffer and answers 1984 IDW queries.  Reports p50/p99 of the
per-cycle latency (device events and host wall clock) and spot-checks parity against the
CPU oracle (which replays the same deltas) at chosen cycles.

    python tools/config_e.py [--cycles 200] [--check 0,100,199] [--out gpurun_out/config_e.json]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_2503_22588_b200 as nbt
from nbt_inputs import CONFIGS, FOV_H, FOV_V, cycle_deltas, query_points


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cycles", type=int, default=200)
    ap.add_argument("--check", default="0,100,199")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    cfg = CONFIGS["E"]
    checks = {int(c) for c in args.check.split(",") if c}
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    torch.cuda.set_stream(st)
    ctx = nbt.Ctx(0, st.cuda_stream)
    codes = cfg.map_codes()
    m = nbt.Map(ctx, nbt.map_desc(cfg.n, cfg.n, cfg.n, cfg.voxel_size))
    m.upload(codes)
    host_codes = codes.copy()                  # the map as the sensor side knows it
    cam = nbt.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
    n_b, n_q, p = cfg.extra["n_b"], cfg.extra["queries"], cfg.extra["power_p"]
    buf = nbt.IdBuffer(ctx, n_b, cfg.n_persp)
    persp = torch.empty((cfg.n_persp, 3), dtype=torch.float64, device=dev)
    cloud = nbt.empty_cloud(cfg.n_persp, device=dev)
    q_out = torch.empty(n_q, dtype=torch.float64, device=dev)
    poi0 = cfg.poi
    dev_ms, wall_ms, parity = [], [], []
    for t in range(args.cycles):
        ang = 2 * math.pi * t / 200.0
        poi = poi0 + 10 * cfg.voxel_size * np.array([math.cos(ang), math.sin(ang), 0.0])
        poi_vox = (poi / cfg.voxel_size).tolist()
        ijk, vals = cycle_deltas(cfg.n, poi_vox, t, host_codes, seed=cfg.persp_seed)
        host_codes[ijk[:, 2], ijk[:, 1], ijk[:, 0]] = vals     # in order: last delta wins
        q = torch.from_numpy(query_points(n_q, poi, cfg.persp_radius, 0.5, 1.2, seed=t)).to(dev)
        d_ijk, d_val = torch.from_numpy(ijk).to(dev), torch.from_numpy(vals).to(dev)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        e0.record(st)
        m.update(d_ijk, d_val)
        nbt.sample_perspectives(ctx, poi, cfg.persp_radius, cfg.n_persp, cfg.persp_seed + t, cfg.persp_mode, out=persp)
        nbt.id_compute(ctx, m, poi, persp, cam, cfg.range_, out=cloud)
        buf.push(cloud, cfg.n_persp)
        buf.query(q, power_p=p, out=q_out)
        e1.record(st)
        ctx.sync()
        wall_ms.append(1e3 * (time.perf_counter() - w0))
        dev_ms.append(e0.elapsed_time(e1))
        if t in checks:
            import oracle
            om = oracle.OracleMap(host_codes, voxel_size=cfg.voxel_size)
            ocam = oracle.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
            P = persp.cpu().numpy()
            _, g, c = oracle.id_compute(om, poi, P, ocam, cfg.range_, nthreads=os.cpu_count() or 1)
            ok_counts = bool(np.array_equal(cloud.counts.cpu().numpy().astype(np.int64), c))
            ok_gain = bool(np.array_equal(cloud.gain.cpu().numpy(), g))
            ok_map = bool(np.array_equal(m.download(), host_codes))
            parity.append({"cycle": t, "map_equal": ok_map, "counts_equal": ok_counts, "gain_equal": ok_gain})
    res = {"config": "E: 256^3 SYN map, 512 perspectives x 64x48 rays per cycle, moving PoI, map deltas, "
                     f"N_B={n_b}, {n_q} IDW queries per cycle", "cycles": args.cycles,
           "device_ms_p50": float(np.percentile(dev_ms[1:], 50)), "device_ms_p99": float(np.percentile(dev_ms[1:], 99)),
           "wall_ms_p50": float(np.percentile(wall_ms[1:], 50)), "wall_ms_p99": float(np.percentile(wall_ms[1:], 99)),
           "parity": parity}
    print(json.dumps(res))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)
    assert all(r["map_equal"] and r["counts_equal"] and r["gain_equal"] for r in parity), parity


if __name__ == "__main__":
    main()
