"""Config E: the receding-horizon loop.  200 MHP cycles; each cycle applies
that cycle's map deltas, samples 512 perspectives around a moving PoI, recomputes the ID,
pushes it into the N_B = 10 buffer and answers 1984 IDW queries.  Reports p50/p99 of the
per-cycle latency (device events and host wall clock).  Oracle parity of the loop (map
replica, totals, g_P, IDW values) is checked by tests/test_gpu_parity.py through run_loop's
callback; this tool itself never touches the oracle.

    python tools/config_e.py [--cycles 200] [--out gpurun_out/config_e.json]
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


def run_loop(cycles, on_cycle=None):
    """Run the config E loop; on_cycle(t, state) is called after each cycle with the
    device results (used by tests for oracle parity).  Returns per-cycle device/wall ms."""
    cfg = CONFIGS["E"]
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
    dev_ms, wall_ms = [], []
    for t in range(cycles):
        ang = 2 * math.pi * t / 200.0
        poi = cfg.poi + 10 * cfg.voxel_size * np.array([math.cos(ang), math.sin(ang), 0.0])
        poi_vox = (poi / cfg.voxel_size).tolist()
        ijk, vals = cycle_deltas(cfg.n, poi_vox, t, host_codes, seed=cfg.persp_seed)
        host_codes[ijk[:, 2], ijk[:, 1], ijk[:, 0]] = vals     # in order: last delta wins
        q_host = query_points(n_q, poi, cfg.persp_radius, 0.5, 1.2, seed=t)
        q = torch.from_numpy(q_host).to(dev)
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
        if on_cycle is not None:
            on_cycle(t, {"cfg": cfg, "poi": poi, "codes": host_codes, "map": m, "persp": persp, "cloud": cloud,
                         "cam": cam, "queries": q_host, "idw": q_out})
    return dev_ms, wall_ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cycles", type=int, default=200)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev_ms, wall_ms = run_loop(args.cycles)
    res = {"config": "E: 256^3 SYN map, 512 perspectives x 64x48 rays per cycle, moving PoI, map deltas, "
                     "N_B=10, 1984 IDW queries per cycle", "cycles": args.cycles,
           "device_ms_p50": float(np.percentile(dev_ms[1:], 50)), "device_ms_p99": float(np.percentile(dev_ms[1:], 99)),
           "wall_ms_p50": float(np.percentile(wall_ms[1:], 50)), "wall_ms_p99": float(np.percentile(wall_ms[1:], 99)),
           "parity": "checked by tests/test_gpu_parity.py::test_config_e_loop (cycles 0, 100, 199)"}
    print(json.dumps(res))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
