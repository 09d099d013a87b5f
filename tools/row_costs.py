"""Walk cost per 8x4 tile position of the camera lattice (the order in which the trace hands out its
work chunks matters at the end of a launch): per-ray in-grid lookups of the
production trace kernel (nbt_debug_id_rays) averaged over a config's perspectives, reported per tile
row (mean and the mean of each tile's longest ray, the lockstep walk's cost) and per tile column.

    python tools/row_costs.py B [D ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np

import paper_2503_22588_b200 as nbt
from nbt_inputs import CONFIGS, FOV_H, FOV_V


def main():
    ctx = nbt.Ctx(0)
    for name in sys.argv[1:] or ["B"]:
        cfg = CONFIGS[name]
        m = nbt.Map(ctx, nbt.map_desc(cfg.n, cfg.n, cfg.n, cfg.voxel_size))
        m.upload(cfg.map_codes())
        cam = nbt.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
        P = nbt.sample_perspectives(ctx, cfg.poi, cfg.persp_radius, cfg.n_persp, cfg.persp_seed, cfg.persp_mode)
        P = np.asarray(P)[:: max(1, cfg.n_persp // 256)]
        rec = nbt.debug_id_rays(ctx, m, cfg.poi, P, cam, cfg.range_)
        look = rec[:, : cfg.width * cfg.height, 3].astype(np.float64).reshape(len(P), cfg.height, cfg.width)
        th, tw = cfg.height // 4, cfg.width // 8
        tiles = look[:, : th * 4, : tw * 8].reshape(len(P), th, 4, tw, 8)
        mean_t = tiles.mean(axis=(2, 4)).mean(axis=0)            # [th, tw]
        max_t = tiles.max(axis=(2, 4)).mean(axis=0)              # lockstep cost ~ longest ray
        print(json.dumps({"config": name, "perspectives": len(P),
                          "row_mean": [round(x, 1) for x in mean_t.mean(axis=1)],
                          "row_tile_max": [round(x, 1) for x in max_t.mean(axis=1)],
                          "col_tile_max": [round(x, 1) for x in max_t.mean(axis=0)]}), flush=True)
        m.close()


if __name__ == "__main__":
    main()
