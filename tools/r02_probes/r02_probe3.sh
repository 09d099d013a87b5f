# round 2: GPU suite, the re-anchored bench (config D headline), and a world-2 gloo run of the
# strong-scaling path on the one GPU (checksums must equal the N = 1 line)
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests3.log 2>&1
tail -5 gpurun_out/gpu_tests3.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench3.json 2> gpurun_out/bench3.err
tail -3 gpurun_out/bench3.err
NBT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 6 --warmup 3 --no-cpu-baseline --no-integrate --no-north-star --no-config-b > gpurun_out/bench3_w2.json 2> gpurun_out/bench3_w2.err
tail -3 gpurun_out/bench3_w2.err
