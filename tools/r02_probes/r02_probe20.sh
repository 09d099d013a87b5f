# round 2: IDW lanes-per-query-group (8/16/32) and queries per thread (3/4) on the fused kernel
set -x
for lib in libnbt.so variants/libnbt_isp32.so variants/libnbt_isp32q4.so variants/libnbt_isp8.so variants/libnbt_iq4.so; do NBT_LIB=paper_2503_22588_b200/$lib python tools/idw_probe.py >> gpurun_out/idw20.log 2>&1; done
python -c "
import sys, json
for l in open('gpurun_out/idw20.log'):
    try: d=json.loads(l)
    except Exception: continue
    print(d['lib'], d['n_persp'], round(d['us_p50'],1), round(d['us_min'],1), d['checksum'])
"
