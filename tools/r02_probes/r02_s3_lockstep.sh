# round 2 session 3: tile-lockstep (refill only when all 32 lanes are idle) -- tile shapes and batch sizes under it
set -x
for i in 1 2; do
for lib in libnbt.so variants/libnbt_tile4.so variants/libnbt_tile16.so variants/libnbt_k12.so variants/libnbt_k8.so; do
  echo "== $lib refill 32" >> gpurun_out/s3_lockstep.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 10 --opt TRACE_REFILL_MIN=32 >> gpurun_out/s3_lockstep.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 10 --opt TRACE_REFILL_MIN=32 >> gpurun_out/s3_lockstep.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s3_lockstep.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
