# round 2 session 4: measurement pass after the byte-store load change -- driver bench line, its ncu launch list,
# ncu --set full of k_id_trace on D / C' (byte) / B and of the IDW query, world-2 gloo checksum run
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s4b_bench.json 2> gpurun_out/s4b_bench.err; tail -2 gpurun_out/s4b_bench.err
python bench.py --gpus 1 --steps 6 --warmup 3 --no-cpu-baseline --no-integrate --no-north-star --no-config-b --no-config-e --no-e2e > gpurun_out/s4b_bench_s6.json 2>&1
NBT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 6 --warmup 3 --no-cpu-baseline --no-integrate --no-north-star --no-config-b --no-config-e > gpurun_out/s4b_bench_w2.json 2> gpurun_out/s4b_bench_w2.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/s4b_launches.csv python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s4b_ncu_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/s4b_trace_d python tools/trace_variants.py D --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/s4b_trace_cp8 python tools/trace_variants.py "C'" --bits 8 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/s4b_trace_b python tools/trace_variants.py B --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_idw -s 3 -c 1 -o gpurun_out/s4b_idw python tools/idw_probe.py > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
