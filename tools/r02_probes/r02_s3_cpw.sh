# round 2 session 3: chunk size aimed at 4 / 8 / 16 chunks per resident warp (B's tail: 32-slot chunks), with CHUNK_MIN 32
set -x
for i in 1 2; do
for lib in libnbt.so variants/libnbt_cpw8.so variants/libnbt_cpw16.so; do
  echo "== $lib" >> gpurun_out/s3_cpw.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 10 --opt TRACE_CHUNK_MIN=32 >> gpurun_out/s3_cpw.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B --reps 10 >> gpurun_out/s3_cpw.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s3_cpw.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
