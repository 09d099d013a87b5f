"""End-to-end time of row f3 from host numpy frames (staging + H2D + kernels + the counters'
D2H), config F, 8 frames x 8 repetitions; also a plain numpy copy of one frame for the host's
memory-copy speed.  Used for the copy-thread measurements (profiles/r01_h2d_copy_threads.log);
the ctx option NBT_OPT_COPY_THREADS is the first argument (0 or 1, default 1):
    python tools/e2e_integrate_probe.py 1
"""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_22588_b200 as nbt
from nbt_inputs import CLOUD_CONFIGS
cf = CLOUD_CONFIGS["F"]
dev = torch.device("cuda", 0)
s = torch.cuda.Stream(dev); torch.cuda.set_stream(s)
ctx = nbt.Ctx(0, s.cuda_stream)
COPY = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ctx.set_option(nbt.OPT_COPY_THREADS, COPY)
desc = nbt.map_desc(cf.n, cf.n, cf.n, cf.voxel_size)
occ = nbt.OccMap(ctx, desc); mi = nbt.Map(ctx, desc)
prm = nbt.integrate_params(cf.voxel_size, leaf=cf.leaf, max_range=cf.max_range)
clouds = [cf.cloud(k) for k in range(cf.n_clouds)]
occ.integrate(cf.sensor(0), clouds[0], map=mi, params=prm); occ.stats()
ts = []
for rep in range(8):
    for k in range(cf.n_clouds):
        t0 = time.perf_counter()
        occ.integrate(cf.sensor(k), clouds[k], map=mi, params=prm)
        occ.stats()
        ts.append(1e3 * (time.perf_counter() - t0))
dst = np.empty((max(len(c) for c in clouds), 3))
mc = []
for rep in range(20):
    t0 = time.perf_counter(); c = clouds[rep % cf.n_clouds]; np.copyto(dst[:len(c)], c); mc.append(1e3 * (time.perf_counter() - t0))
print(f"copy_threads={COPY}", "e2e ms/frame min %.3f p50 %.3f mean %.3f | numpy 8.8MB copy p50 %.3f ms" % (
    min(ts), statistics.median(ts), statistics.mean(ts), statistics.median(mc)))
