# round 2 session 3: lockstep instance (queue-free, one-vote exit) -- GPU suite, 2000 fuzz configurations, A/B vs HEAD
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3_lock3_tests.log 2>&1; tail -2 gpurun_out/s3_lock3_tests.log
NBT_FUZZ_SEEDS=1000 timeout 900 python -m pytest tests -m gpu -k fuzz -q 2>&1 | tail -1
for i in 1 2; do
for lib in variants/libnbt_head.so libnbt.so; do
  echo "== $lib" >> gpurun_out/s3_lock3.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 10 >> gpurun_out/s3_lock3.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 10 >> gpurun_out/s3_lock3.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s3_lock3.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
