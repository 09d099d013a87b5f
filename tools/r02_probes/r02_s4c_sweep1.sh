# round 2 session 4: register budget (3 / 4 / 5 blocks per SM) on the final build -- A/B
set -x
for i in 1 2; do
for lib in libnbt.so variants/libnbt_minb5.so variants/libnbt_minb3.so; do
  echo "== $lib" >> gpurun_out/s4c_sweep1.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 8 >> gpurun_out/s4c_sweep1.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 5 >> gpurun_out/s4c_sweep1.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s4c_sweep1.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['persp'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
