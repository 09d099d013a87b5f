# round 2: multi-rank functional runs of the strong-scaling bench on the one GPU (gloo): world 3
# (uneven shards and query slices) and world 2 with the peer-memory gather; checksums vs N = 1
set -x
python bench.py --gpus 1 --steps 4 --warmup 3 --no-cpu-baseline --no-integrate --no-north-star --no-config-b --no-config-e --no-e2e > gpurun_out/w1.json 2>&1
NBT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 3 --steps 4 --warmup 3 --no-cpu-baseline --no-integrate --no-north-star --no-config-b --no-config-e > gpurun_out/w3.json 2> gpurun_out/w3.err
NBT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus 2 --steps 4 --warmup 3 --gather p2p --no-cpu-baseline --no-integrate --no-north-star --no-config-b --no-config-e > gpurun_out/w2p.json 2> gpurun_out/w2p.err
for f in w1 w3 w2p; do python -c "
import json
d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1])
print('$f', d['n_gpus'], round(d['value']/1e9,3), d['config']['parallelism'], json.dumps(d['checksum']))
"; done
tail -3 gpurun_out/w3.err gpurun_out/w2p.err
