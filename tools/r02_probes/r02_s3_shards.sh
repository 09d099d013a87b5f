# round 2 session 3: one rank's strided shard of D (N = 2 / 4 / 8: 2048 / 1024 / 512 perspectives) -- chunk sizing for mid-size launches
set -x
for i in 1 2; do
for lib in libnbt.so variants/libnbt_cpw16.so variants/libnbt_cpw32.so; do
  echo "== $lib" >> gpurun_out/s3_shards.log
  for s in 2 4 8; do NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py D --reps 10 --persp $((4096 / s)) --stride $s >> gpurun_out/s3_shards.log 2>&1; done
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 10 >> gpurun_out/s3_shards.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 6 >> gpurun_out/s3_shards.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s3_shards.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['persp'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
