# round 2 session 3: measurement pass on the current build -- driver bench line, ncu --set full of k_id_trace on D / C' (byte) / B
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; tail -2 gpurun_out/s3_bench.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/s3_trace_d python tools/trace_variants.py D --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/s3_trace_cp8 python tools/trace_variants.py "C'" --bits 8 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/s3_trace_b python tools/trace_variants.py B --reps 1 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
