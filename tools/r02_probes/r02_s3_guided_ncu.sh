# round 2 session 3: ncu of C' (byte store) with guided units vs fixed chunks (why the guided build is slower there)
set -x
timeout 600 ncu --set full --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/s3g_cp8_guided python tools/trace_variants.py "C'" --bits 8 --reps 1 > /dev/null 2>&1
NBT_LIB=paper_2503_22588_b200/variants/libnbt_fixedchunk.so timeout 600 ncu --set full --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/s3g_cp8_fixed python tools/trace_variants.py "C'" --bits 8 --reps 1 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
