# round 2: step-table DDA variant vs the default build, 2-bit and byte stores
set -x
python tools/trace_variants.py B "C'" D > gpurun_out/tv4_base.log 2>&1
NBT_LIB=paper_2503_22588_b200/variants/libnbt_tab.so python tools/trace_variants.py B "C'" D > gpurun_out/tv4_tab.log 2>&1
NBT_LIB=paper_2503_22588_b200/variants/libnbt_tab.so python tools/trace_variants.py B "C'" --bits 8 > gpurun_out/tv4_tab_bytes.log 2>&1
cat gpurun_out/tv4_*.log
NBT_LIB=paper_2503_22588_b200/variants/libnbt_tab.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/tab_cp python tools/trace_variants.py "C'" --reps 1 > /dev/null 2>&1
NBT_LIB=paper_2503_22588_b200/variants/libnbt_tab.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/tab_d python tools/trace_variants.py D --reps 1 > /dev/null 2>&1
ls gpurun_out
