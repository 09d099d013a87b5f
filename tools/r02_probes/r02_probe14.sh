# round 2: full GPU suite (incl. the full-size per-ray parity of the production trace)
set -x
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests14.log 2>&1; tail -5 gpurun_out/gpu_tests14.log
python -m pytest tests -m gpu -q -k "full_size" --durations=5 >> gpurun_out/gpu_tests14.log 2>&1; tail -12 gpurun_out/gpu_tests14.log
