# round 2 session 3: ncu --set full of k_id_trace on D / C' (byte) / B under tile lockstep (default)
set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/s3l_trace_d python tools/trace_variants.py D --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/s3l_trace_cp8 python tools/trace_variants.py "C'" --bits 8 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/s3l_trace_b python tools/trace_variants.py B --reps 1 > /dev/null 2>&1
ls gpurun_out/s3l_*.ncu-rep
