# round 2 session 4: GPU suite + 3000-seed fuzz, then the measurement pass (tag s4c) of the build with bank-padded rows / planes, the 2-bit word address on the ALU pipe and the per-store x-first predicate
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s4c_gpu_tests.log 2>&1; tail -2 gpurun_out/s4c_gpu_tests.log
NBT_FUZZ_SEEDS=3000 timeout 1500 python -m pytest tests -m gpu -k fuzz -q > gpurun_out/s4c_gpu_fuzz3000.log 2>&1; tail -2 gpurun_out/s4c_gpu_fuzz3000.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s4c_smoke.log 2>&1; tail -1 gpurun_out/s4c_smoke.log
# ncu --set full of k_id_trace on D / C' (byte) / B and of the IDW query, world-2 gloo checksum run
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s4c_bench.json 2> gpurun_out/s4c_bench.err; tail -2 gpurun_out/s4c_bench.err
python bench.py --gpus 1 --steps 6 --warmup 3 --no-cpu-baseline --no-integrate --no-north-star --no-config-b --no-config-e --no-e2e > gpurun_out/s4c_bench_s6.json 2>&1
NBT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 6 --warmup 3 --no-cpu-baseline --no-integrate --no-north-star --no-config-b --no-config-e > gpurun_out/s4c_bench_w2.json 2> gpurun_out/s4c_bench_w2.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/s4c_launches.csv python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s4c_ncu_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/s4c_trace_d python tools/trace_variants.py D --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/s4c_trace_cp8 python tools/trace_variants.py "C'" --bits 8 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/s4c_trace_b python tools/trace_variants.py B --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_idw -s 3 -c 1 -o gpurun_out/s4c_idw python tools/idw_probe.py > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
