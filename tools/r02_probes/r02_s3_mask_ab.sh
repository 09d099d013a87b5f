# round 2 session 3: same-session A/B of the DDA step's 0/1-flag form (HEAD build) vs the 0/-1-mask form (current build)
set -x
for i in 1 2 3; do
for lib in variants/libnbt_head.so libnbt.so; do
  echo "== $lib" >> gpurun_out/s3_mask_ab.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 10 >> gpurun_out/s3_mask_ab.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 10 >> gpurun_out/s3_mask_ab.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s3_mask_ab.log'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print(' ', d['config'], d['store'], round(d['trace_ms'],4), d['checksum'])
"
