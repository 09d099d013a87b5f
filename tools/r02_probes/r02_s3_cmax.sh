# round 2 session 3: largest work chunk 1024 / 512 / 256 slots under tile lockstep (the end-of-launch tail of D and C')
set -x
for i in 1 2; do
for lib in variants/libnbt_cmax256.so variants/libnbt_cmax128.so variants/libnbt_cmax64.so; do
  echo "== $lib" >> gpurun_out/s3_cmax2.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 10 >> gpurun_out/s3_cmax2.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 10 >> gpurun_out/s3_cmax2.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s3_cmax2.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
