# round 2 measurement pass: the driver's bench command, its ncu launch list, one ncu --set full of
# k_id_trace on D (2-bit) and C' (byte store), and a world-2 gloo run (checksum vs N = 1)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -2 gpurun_out/final_bench.err
python bench.py --gpus 1 --steps 6 --warmup 3 --no-cpu-baseline --no-integrate --no-north-star --no-config-b --no-config-e --no-e2e > gpurun_out/final_bench_s6.json 2>&1
NBT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 6 --warmup 3 --no-cpu-baseline --no-integrate --no-north-star --no-config-b --no-config-e > gpurun_out/final_bench_w2.json 2> gpurun_out/final_bench_w2.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/final_launches.csv python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/final_ncu_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/final_trace_d python tools/trace_variants.py D --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/final_trace_cp8 python tools/trace_variants.py "C'" --bits 8 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/final_trace_b python tools/trace_variants.py B --reps 1 > /dev/null 2>&1
ls -la gpurun_out
