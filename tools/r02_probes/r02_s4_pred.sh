# round 2 session 4: the DDA step as predicates + predicated adds (dda.cuh NBT_DDA_PRED=1) against the flag form -- A/B
set -x
./build/dda_step_forms > gpurun_out/s4_step_forms.log 2>&1
for i in 1 2; do
for lib in variants/libnbt_flagstep.so libnbt.so; do
  echo "== $lib" >> gpurun_out/s4_pred.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 10 >> gpurun_out/s4_pred.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 6 >> gpurun_out/s4_pred.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s4_pred.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['persp'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
cat gpurun_out/s4_step_forms.log
