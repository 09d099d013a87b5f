# round 2 session 4: GPU suite + 3000-seed ID / integration fuzz on the predicated DDA step
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4_gpu_tests.log 2>&1; tail -2 gpurun_out/s4_gpu_tests.log
NBT_FUZZ_SEEDS=3000 timeout 1500 python -m pytest tests -m gpu -k fuzz -q > gpurun_out/s4_gpu_fuzz3000.log 2>&1; tail -2 gpurun_out/s4_gpu_fuzz3000.log
