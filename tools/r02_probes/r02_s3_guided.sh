# round 2 session 3: guided self-scheduling of 32-ray work units (shrinking grabs) vs fixed chunks -- GPU suite + A/B
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3_guided_tests.log 2>&1; tail -3 gpurun_out/s3_guided_tests.log
for i in 1 2; do
for lib in variants/libnbt_fixedchunk.so libnbt.so; do
  echo "== $lib" >> gpurun_out/s3_guided.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 10 >> gpurun_out/s3_guided.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 10 >> gpurun_out/s3_guided.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s3_guided.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
