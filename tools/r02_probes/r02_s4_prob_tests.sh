# round 2 session 4: GPU suite + 1000-seed fuzz after the f1 byte-load change (the first suite run stopped on a host-timing bound)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s4_prob_tests2.log 2>&1; tail -2 gpurun_out/s4_prob_tests2.log
NBT_FUZZ_SEEDS=1000 timeout 1500 python -m pytest tests -m gpu -k fuzz -q > gpurun_out/s4_prob_fuzz1000.log 2>&1; tail -2 gpurun_out/s4_prob_fuzz1000.log
