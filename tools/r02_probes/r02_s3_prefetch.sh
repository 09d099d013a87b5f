# round 2 session 3: chunk grab prefetched one chunk ahead, perspective status checked per ray -- GPU suite + A/B (also 32-slot chunks on B)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3_pf_tests.log 2>&1; tail -3 gpurun_out/s3_pf_tests.log
for i in 1 2; do
for lib in variants/libnbt_head.so libnbt.so; do
  echo "== $lib" >> gpurun_out/s3_prefetch.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 10 >> gpurun_out/s3_prefetch.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 10 >> gpurun_out/s3_prefetch.log 2>&1
done
echo "== cpw8 chunk 32 (B)" >> gpurun_out/s3_prefetch.log
NBT_LIB=paper_2503_22588_b200/variants/libnbt_cpw8.so python tools/trace_variants.py B --reps 20 --opt TRACE_CHUNK_MIN=32 >> gpurun_out/s3_prefetch.log 2>&1
done
python -c "
import json
for l in open('gpurun_out/s3_prefetch.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
