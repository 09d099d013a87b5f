"""Measure how long neighbouring rays of a perspective walk the SAME voxel sequence (the premise
of beam / packet traversal for dense lattices, verdict r01 lever (a)): on config C' (640x480 rays,
256^3 SYN map) and D (160x120, 512^3), the oracle's walk of every ray of random 8x4 pixel tiles;
report the mean ray length (visits until the stop or the end), the mean common prefix of
horizontally adjacent rays, and the prefix shared by all 32 rays of the tile.  Oracle only, CPU.

    python tests/analysis/beam_prefix.py [--tiles 60] [--persp 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np

import oracle
from nbt_inputs import CONFIGS, FOV_H, FOV_V


def prefix(a, b):
    n = min(len(a), len(b))
    k = 0
    while k < n and a[k] == b[k]:
        k += 1
    return k


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tiles", type=int, default=60)
    ap.add_argument("--persp", type=int, default=3)
    args = ap.parse_args()
    rng = np.random.default_rng(0)
    out = []
    for name in ("C'", "D"):
        cfg = CONFIGS[name]
        om = oracle.OracleMap(cfg.map_codes(), voxel_size=cfg.voxel_size)
        cam = oracle.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
        P = oracle.sample_perspectives(cfg.poi, cfg.persp_radius, cfg.n_persp, cfg.persp_seed, cfg.persp_mode)
        lens, adj, tile_pref = [], [], []
        for p in P[:: max(1, cfg.n_persp // args.persp)][: args.persp]:
            o, e, _ = oracle.perspective_rays(om, cfg.poi, p, cam, cfg.range_, with_counts=False)
            for _ in range(args.tiles):
                tx = int(rng.integers(0, cfg.width // 8)) * 8
                ty = int(rng.integers(0, cfg.height // 4)) * 4
                seqs = []
                for kk in range(ty, ty + 4):
                    row = []
                    for i in range(tx, tx + 8):
                        k = kk * cfg.width + i
                        ijk, _, r = oracle.trace_ray(om, o, e[k], max_visits=4096)
                        s = [tuple(v) for v in ijk]
                        row.append(s)
                        lens.append(len(s))
                    for a, b in zip(row, row[1:]):
                        adj.append(prefix(a, b))
                    seqs.extend(row)
                tp = min(prefix(seqs[0], s) for s in seqs[1:])
                tile_pref.append(tp)
        res = {"config": name, "rays": len(lens), "mean_visits": float(np.mean(lens)),
               "adjacent_common_prefix_mean": float(np.mean(adj)),
               "adjacent_prefix_share": float(np.sum(adj) / np.sum(lens)),
               "tile32_common_prefix_mean": float(np.mean(tile_pref)),
               "tile32_prefix_share": float(np.mean(tile_pref) / np.mean(lens))}
        print(json.dumps(res), flush=True)
        out.append(res)


if __name__ == "__main__":
    main()
