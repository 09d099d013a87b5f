# round 2 session 3: baseline on a fresh box -- GPU suite, trace times B / C' (byte) / D
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3_gpu_tests.log 2>&1; tail -3 gpurun_out/s3_gpu_tests.log
for i in 1 2; do python tools/trace_variants.py B "C'" D --reps 10 >> gpurun_out/s3_base_trace.log 2>&1; python tools/trace_variants.py "C'" --bits 8 --reps 10 >> gpurun_out/s3_base_trace.log 2>&1; done
cat gpurun_out/s3_base_trace.log
