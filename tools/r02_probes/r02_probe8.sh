# round 2: persistent IDW variants; trace refill / chunk retune on D and C'
set -x
for lib in libnbt.so variants/libnbt_oldidw.so variants/libnbt_pmb2.so variants/libnbt_pmb8.so variants/libnbt_pq2.so variants/libnbt_plb3.so; do NBT_LIB=paper_2503_22588_b200/$lib python tools/idw_probe.py >> gpurun_out/idw8.log 2>&1; done
python -c "
import sys, json
for l in open('gpurun_out/idw8.log'):
    try: d=json.loads(l)
    except Exception: continue
    print(d['lib'], d['n_persp'], round(d['us_p50'],1), round(d['us_min'],1), d['checksum'])
"
for o in "" "--opt TRACE_REFILL_MIN=3" "--opt TRACE_REFILL_MIN=12" "--opt TRACE_REFILL_MIN=20" "--opt TRACE_CHUNK_MIN=256" "--opt TRACE_CHUNK_MIN=1024"; do echo "== $o"; python tools/trace_variants.py D $o; done > gpurun_out/tv8_d.log 2>&1
cat gpurun_out/tv8_d.log | cut -c1-120
ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_idw python tools/idw_probe.py > gpurun_out/idw8_ncu.log 2>&1
grep -E "k_idw|duration|warps_active|fp64|issue_active" gpurun_out/idw8_ncu.log | head -40
