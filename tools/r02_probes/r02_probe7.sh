# round 2: IDW register-budget / chunking variants, DFMA peak, full GPU suite
set -x
./build/peaks > gpurun_out/peaks7.json 2>&1; grep -E "dfma|int32_peak_tops" gpurun_out/peaks7.json
for lib in libnbt.so variants/libnbt_oldidw.so variants/libnbt_lb3mb1.so variants/libnbt_lb3mb3.so variants/libnbt_lb4mb4.so variants/libnbt_lb4q2mb4.so variants/libnbt_lb4q2mb8.so; do NBT_LIB=paper_2503_22588_b200/$lib python tools/idw_probe.py >> gpurun_out/idw7.log 2>&1; done
cat gpurun_out/idw7.log
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests7.log 2>&1; tail -5 gpurun_out/gpu_tests7.log
