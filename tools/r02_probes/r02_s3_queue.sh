# round 2 session 3: packed prepared-walk queue (int2 columns, no per-ray perspective / pre), int lane flag -- GPU suite + A/B vs HEAD
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3_queue3_tests.log 2>&1; tail -3 gpurun_out/s3_queue3_tests.log
for i in 1 2; do
for lib in variants/libnbt_head.so libnbt.so; do
  echo "== $lib" >> gpurun_out/s3_queue3.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 10 >> gpurun_out/s3_queue3.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 10 >> gpurun_out/s3_queue3.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s3_queue3.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
