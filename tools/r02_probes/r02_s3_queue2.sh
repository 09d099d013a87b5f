# round 2 session 3: C' byte store after the packed queue: mask vs flag step form (HEAD build for reference)
set -x
for i in 1 2 3; do
for lib in variants/libnbt_head.so libnbt.so variants/libnbt_bytflags.so; do
  echo "== $lib" >> gpurun_out/s3_queue2.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 10 >> gpurun_out/s3_queue2.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s3_queue2.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
