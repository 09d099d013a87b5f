# round 2 session 3: tile-lockstep instance (no queue, no shared memory, carveout 0) vs HEAD's per-lane refill (threshold 6)
# and vs HEAD's queue path at threshold 32 -- GPU suite + A/B
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3_lock_tests.log 2>&1; tail -3 gpurun_out/s3_lock_tests.log
for i in 1 2; do
  echo "== head refill 6" >> gpurun_out/s3_lockstep2.log
  NBT_LIB=paper_2503_22588_b200/variants/libnbt_head.so python tools/trace_variants.py B D --reps 10 >> gpurun_out/s3_lockstep2.log 2>&1
  NBT_LIB=paper_2503_22588_b200/variants/libnbt_head.so python tools/trace_variants.py "C'" --bits 8 --reps 10 >> gpurun_out/s3_lockstep2.log 2>&1
  echo "== head queue refill 32" >> gpurun_out/s3_lockstep2.log
  NBT_LIB=paper_2503_22588_b200/variants/libnbt_head.so python tools/trace_variants.py B D --reps 10 --opt TRACE_REFILL_MIN=32 >> gpurun_out/s3_lockstep2.log 2>&1
  NBT_LIB=paper_2503_22588_b200/variants/libnbt_head.so python tools/trace_variants.py "C'" --bits 8 --reps 10 --opt TRACE_REFILL_MIN=32 >> gpurun_out/s3_lockstep2.log 2>&1
  echo "== lockstep instance" >> gpurun_out/s3_lockstep2.log
  python tools/trace_variants.py B D --reps 10 >> gpurun_out/s3_lockstep2.log 2>&1
  python tools/trace_variants.py "C'" --bits 8 --reps 10 >> gpurun_out/s3_lockstep2.log 2>&1
  echo "== lockstep instance carveout 25" >> gpurun_out/s3_lockstep2.log
  python tools/trace_variants.py B D --reps 10 --opt TRACE_CARVEOUT=-1 >> gpurun_out/s3_lockstep2.log 2>&1
done
python -c "
import json
for l in open('gpurun_out/s3_lockstep2.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
