"""Row f3 workload alone (config F frames into a 256^3 store), for ncu launch lists:
    ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/profile_integrate.py
No oracle; device-resident points; 2 passes over the 8 frames."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_22588_b200 as nbt  # noqa: E402
from nbt_inputs import CLOUD_CONFIGS  # noqa: E402


def main():
    cf = CLOUD_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "F"]
    passes = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = nbt.Ctx(0, stream.cuda_stream)
    desc = nbt.map_desc(cf.n, cf.n, cf.n, cf.voxel_size)
    occ = nbt.OccMap(ctx, desc)
    m = nbt.Map(ctx, desc)
    prm = nbt.integrate_params(cf.voxel_size, leaf=cf.leaf, max_range=cf.max_range)
    clouds = [torch.from_numpy(cf.cloud(k)).to(dev) for k in range(cf.n_clouds)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for p in range(passes):
        e0.record(stream)
        for k in range(cf.n_clouds):
            occ.integrate(cf.sensor(k), clouds[k], map=m, params=prm)
        e1.record(stream)
        torch.cuda.synchronize()
        print(f"pass {p}: {e0.elapsed_time(e1) / cf.n_clouds:.4f} ms/frame", occ.stats(), flush=True)


if __name__ == "__main__":
    main()
