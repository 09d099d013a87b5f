# round 2: the original IDW kernel with register budgets for 3-4 resident blocks per SM
set -x
for lib in libnbt.so variants/libnbt_olb3.so variants/libnbt_oq2lb4.so variants/libnbt_oq2lb3.so variants/libnbt_oq1lb4.so; do NBT_LIB=paper_2503_22588_b200/$lib python tools/idw_probe.py >> gpurun_out/idw10.log 2>&1; done
python -c "
import sys, json
for l in open('gpurun_out/idw10.log'):
    try: d=json.loads(l)
    except Exception: continue
    print(d['lib'], d['n_persp'], round(d['us_p50'],1), round(d['us_min'],1), d['checksum'])
"
for lib in libnbt.so variants/libnbt_oq2lb4.so; do NBT_LIB=paper_2503_22588_b200/$lib ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size --clock-control none -k regex:k_idw -c 2 python tools/idw_probe.py > gpurun_out/idw10_ncu_$(basename $lib .so).log 2>&1; grep -E "duration|warps_active|fp64|issue_active|registers|grid_size" gpurun_out/idw10_ncu_$(basename $lib .so).log; done
