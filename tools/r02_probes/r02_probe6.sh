# round 2: SM-affine chunk order; step table + byte store at 50% carveout; IDW old vs chunked (graph-timed)
set -x
python tools/trace_variants.py B "C'" D > gpurun_out/tv6_base.log 2>&1
NBT_LIB=paper_2503_22588_b200/variants/libnbt_aff.so python tools/trace_variants.py B "C'" D > gpurun_out/tv6_aff.log 2>&1
NBT_LIB=paper_2503_22588_b200/variants/libnbt_tab.so python tools/trace_variants.py "C'" --bits 8 --opt TRACE_CARVEOUT=50 > gpurun_out/tv6_tab_bytes_c50.log 2>&1
python tools/trace_variants.py "C'" --bits 8 > gpurun_out/tv6_bytes.log 2>&1
cat gpurun_out/tv6_*.log
for lib in libnbt.so variants/libnbt_oldidw.so variants/libnbt_idwq2.so variants/libnbt_idwmb8.so variants/libnbt_idwmb2.so; do NBT_LIB=paper_2503_22588_b200/$lib python tools/idw_probe.py >> gpurun_out/idw6.log 2>&1; done
cat gpurun_out/idw6.log
NBT_LIB=paper_2503_22588_b200/variants/libnbt_aff.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/aff_d python tools/trace_variants.py D --reps 1 > /dev/null 2>&1
