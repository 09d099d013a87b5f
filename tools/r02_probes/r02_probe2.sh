# round 2: GPU suite after the Q16 walk / options / record instance, plus store variants of the trace
set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/gpu_tests.log
tail -5 gpurun_out/gpu_tests.log
python tools/trace_variants.py B "C'" D > gpurun_out/tv_q16.log 2>&1
python tools/trace_variants.py B "C'" D --bits 8 > gpurun_out/tv_bytes.log 2>&1
python tools/trace_variants.py B "C'" D --layout morton > gpurun_out/tv_morton.log 2>&1
cat gpurun_out/tv_q16.log gpurun_out/tv_bytes.log gpurun_out/tv_morton.log
