# round 2 session 3: refill threshold (idle lanes before a warp refills) 4 / 6 / 8 / 10 on the session-3 loop
set -x
for i in 1 2; do
for r in 32 28 30 31; do
  echo "== refill $r" >> gpurun_out/s3_refill3.log
  python tools/trace_variants.py B D --reps 10 --opt TRACE_REFILL_MIN=$r >> gpurun_out/s3_refill3.log 2>&1
  python tools/trace_variants.py "C'" --bits 8 --reps 10 --opt TRACE_REFILL_MIN=$r >> gpurun_out/s3_refill3.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s3_refill3.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
