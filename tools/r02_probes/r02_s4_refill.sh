# round 2 session 4: per-lane refill thresholds re-measured on the final build (issue-bound now, L1 75-81%) -- TRACE_REFILL_MIN 32 (lockstep) / 28 / 24 / 16 / 8
set -x
for i in 1 2; do
for r in 32 28 24 16 8; do
  echo "== refill $r" >> gpurun_out/s4_refill.log
  python tools/trace_variants.py B D --reps 6 --opt TRACE_REFILL_MIN=$r >> gpurun_out/s4_refill.log 2>&1
  python tools/trace_variants.py "C'" --bits 8 --reps 4 --opt TRACE_REFILL_MIN=$r >> gpurun_out/s4_refill.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s4_refill.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['persp'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
