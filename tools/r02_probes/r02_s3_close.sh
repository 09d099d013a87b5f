# round 2 session 3: branch-free ray close in batch_finish -- GPU suite + trace times
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3_close_tests.log 2>&1; tail -3 gpurun_out/s3_close_tests.log
for i in 1 2; do python tools/trace_variants.py B "C'" D --reps 10 >> gpurun_out/s3_close_trace.log 2>&1; python tools/trace_variants.py "C'" --bits 8 --reps 10 >> gpurun_out/s3_close_trace.log 2>&1; done
python -c "
import json
for l in open('gpurun_out/s3_close_trace.log'):
    d=json.loads(l); print(d['config'], d['store'], round(d['trace_ms'],4), d['checksum'])
"
