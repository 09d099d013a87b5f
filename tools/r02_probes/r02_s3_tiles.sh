# round 2 session 3: warp tile shape (8x4 default, 4x8, 16x2, 32x1) now that D is L1-data-pipe bound
set -x
for i in 1 2; do
for lib in libnbt.so variants/libnbt_tile4.so variants/libnbt_tile16.so variants/libnbt_tile32.so; do
  echo "== $lib" >> gpurun_out/s3_tiles.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 10 >> gpurun_out/s3_tiles.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 10 >> gpurun_out/s3_tiles.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s3_tiles.log'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print(' ', d['config'], d['store'], round(d['trace_ms'],4), d['checksum'])
"
