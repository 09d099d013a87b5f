set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
./build/peaks > gpurun_out/peaks.json 2> gpurun_out/peaks.err
cat gpurun_out/peaks.json
python tools/trace_variants.py B "C'" D > gpurun_out/tv_base.log 2>&1
cat gpurun_out/tv_base.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/cprime_trace python tools/trace_variants.py "C'" > gpurun_out/ncu_cp.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/d_trace python tools/trace_variants.py D > gpurun_out/ncu_d.log 2>&1
tail -5 gpurun_out/ncu_cp.log
