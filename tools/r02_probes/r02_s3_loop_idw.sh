# round 2 session 3: trace batch loop without the per-batch refill checks (GPU suite + trace times);
# IDW: hardware-reciprocal accuracy, one vs two Newton steps, min d^2 by its high word
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3_loop_tests.log 2>&1; tail -3 gpurun_out/s3_loop_tests.log
for i in 1 2; do python tools/trace_variants.py B "C'" D --reps 10 >> gpurun_out/s3_loop_trace.log 2>&1; python tools/trace_variants.py "C'" --bits 8 --reps 10 >> gpurun_out/s3_loop_trace.log 2>&1; done
cat gpurun_out/s3_loop_trace.log
./build/rcp_probe > gpurun_out/s3_rcp_probe.json; cat gpurun_out/s3_rcp_probe.json
for lib in libnbt.so variants/libnbt_idw_orig.so variants/libnbt_idw_nr1.so variants/libnbt_idw_nr1_q4.so libnbt.so variants/libnbt_idw_nr1.so; do NBT_LIB=paper_2503_22588_b200/$lib python tools/idw_probe.py >> gpurun_out/s3_idw.log 2>&1; done
NBT_LIB=paper_2503_22588_b200/variants/libnbt_idw_nr1.so timeout 600 python -m pytest tests -m gpu -x -q -k "idw or info_cost or smoke" > gpurun_out/s3_idw_nr1_tests.log 2>&1; tail -3 gpurun_out/s3_idw_nr1_tests.log
python -c "
import json
for l in open('gpurun_out/s3_idw.log'):
    try: d=json.loads(l)
    except Exception: continue
    print(d['lib'].split('/')[-1], d['n_persp'], round(d['us_p50'],1), round(d['us_min'],1), d['checksum'])
"
