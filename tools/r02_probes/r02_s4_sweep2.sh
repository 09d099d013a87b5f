# round 2 session 4: D / B are L1-bound again after the predicated step -- tile shape (4x8, 16x2), L1 eviction hints on the map loads, SM-affine chunks (148 homes); step-only ceilings
set -x
./build/dda_step_peak > gpurun_out/s4_step_peak.json 2>&1
for i in 1 2; do
for lib in libnbt.so variants/libnbt_tile4.so variants/libnbt_tile16.so variants/libnbt_load1.so variants/libnbt_load2.so variants/libnbt_affine.so; do
  echo "== $lib" >> gpurun_out/s4_sweep2.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 8 >> gpurun_out/s4_sweep2.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s4_sweep2.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['persp'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
cat gpurun_out/s4_step_peak.json
