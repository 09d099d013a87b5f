# round 2: IDW with the warp-per-query combine; persistent-grid variants
set -x
for lib in libnbt.so variants/libnbt_oldidw.so variants/libnbt_pmb1.so variants/libnbt_pmb2.so variants/libnbt_pq2.so variants/libnbt_pq2mb2.so; do NBT_LIB=paper_2503_22588_b200/$lib python tools/idw_probe.py >> gpurun_out/idw9.log 2>&1; done
python -c "
import sys, json
for l in open('gpurun_out/idw9.log'):
    try: d=json.loads(l)
    except Exception: continue
    print(d['lib'], d['n_persp'], round(d['us_p50'],1), round(d['us_min'],1), d['checksum'])
"
python -m pytest tests -m gpu -x -q -k "idw or info_cost or config_e" > gpurun_out/idw_tests9.log 2>&1; tail -3 gpurun_out/idw_tests9.log
ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size --clock-control none -k regex:k_idw -c 4 python tools/idw_probe.py > gpurun_out/idw9_ncu.log 2>&1
grep -E "k_idw|duration|warps_active|fp64|issue_active|registers|grid_size" gpurun_out/idw9_ncu.log | grep -v PROF | head -40
