# round 2: step table with enough carveout for 4 blocks/SM; IDW chunking variants (timed through tests' shapes)
set -x
for c in 50 62; do NBT_LIB=paper_2503_22588_b200/variants/libnbt_tab.so python tools/trace_variants.py B "C'" D --opt TRACE_CARVEOUT=$c > gpurun_out/tv5_tab_c$c.log 2>&1; done
python tools/trace_variants.py B "C'" D --opt TRACE_CARVEOUT=50 > gpurun_out/tv5_base_c50.log 2>&1
cat gpurun_out/tv5_*.log
for lib in libnbt.so variants/libnbt_idwq2.so variants/libnbt_idwmb8.so variants/libnbt_idwmb2.so; do NBT_LIB=paper_2503_22588_b200/$lib python tools/idw_probe.py >> gpurun_out/idw5.log 2>&1; done
cat gpurun_out/idw5.log
python -m pytest tests -m gpu -x -q -k "idw or info_cost or config_e" > gpurun_out/idw_tests5.log 2>&1; tail -3 gpurun_out/idw_tests5.log
