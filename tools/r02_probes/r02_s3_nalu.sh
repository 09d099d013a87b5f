# round 2 session 3: mask-form DDA step, decision terms on the ALU pipe (NALU) per store kind -- GPU suite + trace times per variant
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3_nalu_tests.log 2>&1; tail -3 gpurun_out/s3_nalu_tests.log
for i in 1 2; do
for lib in libnbt.so variants/libnbt_nalu0.so variants/libnbt_nalub2.so variants/libnbt_nalu2b1.so; do
  echo "== $lib" >> gpurun_out/s3_nalu_trace.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 10 >> gpurun_out/s3_nalu_trace.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 10 >> gpurun_out/s3_nalu_trace.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s3_nalu_trace.log'):
    if l.startswith('=='): print(l.strip()); continue
    d=json.loads(l); print(' ', d['config'], d['store'], round(d['trace_ms'],4), d['checksum'])
"
