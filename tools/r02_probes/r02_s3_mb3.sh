# round 2 session 3: trace register budget for 3 resident blocks (24 warps/SM, up to 80 registers) vs 4 (32 warps, 64)
set -x
for i in 1 2; do
for lib in libnbt.so variants/libnbt_mb3.so; do
  echo "== $lib" >> gpurun_out/s3_mb3.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 10 >> gpurun_out/s3_mb3.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 10 >> gpurun_out/s3_mb3.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s3_mb3.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
