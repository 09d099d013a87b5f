# round 2 session 4: chunk cap 128 / 512, 64 chunks per warp, 4 half chunks at the tail on the final build -- A/B
set -x
for i in 1 2; do
for lib in libnbt.so variants/libnbt_cmax128.so variants/libnbt_cmax512.so variants/libnbt_cpw64.so variants/libnbt_split4.so; do
  echo "== $lib" >> gpurun_out/s4c_chunks.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 8 >> gpurun_out/s4c_chunks.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 5 >> gpurun_out/s4c_chunks.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s4c_chunks.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['persp'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
