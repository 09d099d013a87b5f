# round 2 session 3: IDW warp-per-unit kernel (k_idw_pairs) -- GPU suite, probe vs the block-per-entry form and unit counts
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3_pairs2_tests.log 2>&1; tail -3 gpurun_out/s3_pairs2_tests.log
for lib in libnbt.so variants/libnbt_idw_entry.so variants/libnbt_idw_u4.so variants/libnbt_idw_u16.so libnbt.so; do NBT_LIB=paper_2503_22588_b200/$lib python tools/idw_probe.py >> gpurun_out/s3_pairs2.log 2>&1; done
python -c "
import json
for l in open('gpurun_out/s3_pairs2.log'):
    try: d=json.loads(l)
    except Exception: print(l.rstrip()); continue
    print(d['lib'].split('/')[-1], d['n_persp'], round(d['us_p50'],1), round(d['us_min'],1), d['checksum'])
"
