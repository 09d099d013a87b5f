"""How many distinct 128-B map lines (and 32-B sectors) a lockstep warp request touches -- the
L1 wavefronts per request that bound configs D and B -- for the linear 2-bit store with x
fastest (the store today) and for the same store transposed (y fastest, z fastest), and for a
per-perspective choice of the copy whose fast axis best matches the camera's horizontal axis
(the 8-wide side of a warp's 8x4 tile), and for the Morton store (a 32-B sector = a 4x4x8 block).  The oracle's walk of every ray of random 8x4 tiles;
a request = one visit index of the lockstep walk (all rays of the tile start together), over
the lanes whose ray is still walking inside the grid.  Oracle only, CPU.

    python tests/analysis/line_spread.py [--tiles 40] [--persp 12] [--configs D B]
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

BORDER = 16


def dilate3(v):
    r = np.zeros_like(v)
    for b in range(21):
        r |= ((v >> b) & 1) << (3 * b)
    return r


def bit_offsets(ijk, n, fast):
    """2-bit store bit offsets of voxels ijk (k x 3, x y z) with axis `fast` stored fastest
    (fast = 3: the Morton store, x in the lowest interleaved bit)."""
    if fast == 3:
        v = ijk.astype(np.int64) + BORDER
        return 2 * (dilate3(v[:, 0]) | (dilate3(v[:, 1]) << 1) | (dilate3(v[:, 2]) << 2))
    p = n + 2 * BORDER
    v = ijk.astype(np.int64) + BORDER
    order = {0: (0, 1, 2), 1: (1, 0, 2), 2: (2, 0, 1)}[fast]
    a, b, c = (v[:, order[0]], v[:, order[1]], v[:, order[2]])
    return 2 * (a + p * b + p * p * c)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tiles", type=int, default=40)
    ap.add_argument("--persp", type=int, default=12)
    ap.add_argument("--configs", nargs="+", default=["D", "B"])
    args = ap.parse_args()
    rng = np.random.default_rng(0)
    for name in args.configs:
        cfg = CONFIGS[name]
        om = oracle.OracleMap(cfg.map_codes(), voxel_size=cfg.voxel_size)
        cam = oracle.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
        P = oracle.sample_perspectives(cfg.poi, cfg.persp_radius, cfg.n_persp, cfg.persp_seed, cfg.persp_mode)
        acc = {f: [0, 0, 0] for f in ("x", "y", "z", "morton", "cam", "best")}   # lines, sectors, requests
        for p in P[:: max(1, cfg.n_persp // args.persp)][: args.persp]:
            o, e, _ = oracle.perspective_rays(om, cfg.poi, p, cam, cfg.range_, with_counts=False)
            row = e[(cfg.height // 2) * cfg.width: (cfg.height // 2 + 1) * cfg.width]
            right = np.asarray(row[-1], dtype=np.float64) - np.asarray(row[0], dtype=np.float64)
            cam_fast = int(np.argmax(np.abs(right)))
            per = {f: [0, 0, 0] for f in (0, 1, 2, 3)}
            for _ in range(args.tiles):
                tx = int(rng.integers(0, cfg.width // 8)) * 8
                ty = int(rng.integers(0, cfg.height // 4)) * 4
                walks = []
                for kk in range(ty, ty + 4):
                    for i in range(tx, tx + 8):
                        ijk, codes, _ = oracle.trace_ray(om, o, e[kk * cfg.width + i], max_visits=8192)
                        walks.append(np.asarray(ijk, dtype=np.int64).reshape(-1, 3)[codes != 255])
                steps = max(len(w) for w in walks)
                if steps == 0:
                    continue
                for f in (0, 1, 2, 3):
                    offs = [bit_offsets(w, cfg.n, f) for w in walks]
                    for s in range(steps):
                        b = np.array([o_[s] for o_ in offs if s < len(o_)], dtype=np.int64)
                        per[f][0] += len(np.unique(b >> 10))      # 128-B lines
                        per[f][1] += len(np.unique(b >> 8))       # 32-B sectors
                        per[f][2] += 1
            for f, key in ((0, "x"), (1, "y"), (2, "z"), (3, "morton")):
                for t in range(3):
                    acc[key][t] += per[f][t]
            for t in range(3):
                acc["cam"][t] += per[cam_fast][t]
            bf = min((0, 1, 2), key=lambda f: per[f][0] / max(per[f][2], 1))
            for t in range(3):
                acc["best"][t] += per[bf][t]
        res = {"config": name, "persp": args.persp, "tiles_per_persp": args.tiles}
        for k, (l, s, r) in acc.items():
            res[k] = {"lines_per_request": round(l / max(r, 1), 3), "sectors_per_request": round(s / max(r, 1), 3)}
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
