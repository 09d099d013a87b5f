"""Time the IDW query (row a9, Eq. 4) with a full N_B = 10 buffer: 1984 queries over clouds of
512 (config B/E) and 4096 (config D) perspectives; CUDA events around each query call,
median of 50; NBT_LIB selects a variant build.

    python tools/idw_probe.py
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_2503_22588_b200 as nbt
from nbt_inputs import CONFIGS, query_points

dev = torch.device("cuda", 0)
s = torch.cuda.Stream(dev)
torch.cuda.set_stream(s)
ctx = nbt.Ctx(0, s.cuda_stream)
for n_p in (512, 4096):
    cfg = CONFIGS["B"]
    buf = nbt.IdBuffer(ctx, 10, n_p)
    rng = np.random.default_rng(1)
    for e in range(10):
        xyz = torch.from_numpy(cfg.poi + rng.normal(size=(n_p, 3)) * 0.6).to(dev)
        g = torch.from_numpy(rng.uniform(0, 50, n_p)).to(dev)
        buf.push(nbt.IgCloud(xyz, g, None))
    q = torch.from_numpy(query_points(1984, cfg.poi, cfg.persp_radius, 0.5, 1.2, seed=5)).to(dev)
    out = torch.empty(1984, dtype=torch.float64, device=dev)
    for _ in range(5):
        buf.query(q, out=out)
    ctx.sync()
    ctx.capture_begin()                   # one query call as a graph: no host launch gaps
    buf.query(q, out=out)
    g = ctx.capture_end()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(50):
        e0.record(s)
        g.launch()
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    g.close()
    print(json.dumps({"lib": os.path.basename(os.environ.get("NBT_LIB", "libnbt.so")), "n_persp": n_p,
                      "us_p50": statistics.median(ts), "us_min": min(ts),
                      "pairs_per_s": 1984 * 10 * n_p / (statistics.median(ts) * 1e-6),
                      "checksum": float(out.sum().item())}), flush=True)
    buf.close()
