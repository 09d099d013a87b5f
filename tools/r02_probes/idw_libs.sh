# time the IDW query (tools/idw_probe.py) for each library given: idw_libs.sh LOG LIB...
log=$1; shift
for lib in "$@"; do NBT_LIB=paper_2503_22588_b200/$lib python tools/idw_probe.py >> gpurun_out/$log 2>&1; done
python -c "
import json, sys
for l in open('gpurun_out/$log'):
    try: d=json.loads(l)
    except Exception: print(l.rstrip()); continue
    print(d['lib'].split('/')[-1], d['n_persp'], round(d['us_p50'],1), round(d['us_min'],1), d['checksum'])
"
