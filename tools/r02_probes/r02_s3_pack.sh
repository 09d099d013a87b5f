# round 2 session 3: top-down 2-bit packing (one rotate + one funnel shift per visit) -- GPU suite + trace times
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3_pack_tests.log 2>&1; tail -3 gpurun_out/s3_pack_tests.log
for i in 1 2; do python tools/trace_variants.py B "C'" D --reps 10 >> gpurun_out/s3_pack_trace.log 2>&1; python tools/trace_variants.py "C'" --bits 8 --reps 10 >> gpurun_out/s3_pack_trace.log 2>&1; done
cat gpurun_out/s3_pack_trace.log
