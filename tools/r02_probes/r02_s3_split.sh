# round 2 session 3: the launch's last chunks handed out as halves (NBT_SPLIT_TAIL chunks per warp: 0 / 2 / 4) -- GPU suite + A/B
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3_split_tests.log 2>&1; tail -2 gpurun_out/s3_split_tests.log
for i in 1 2; do
for lib in variants/libnbt_split0.so libnbt.so variants/libnbt_split4.so; do
  echo "== $lib" >> gpurun_out/s3_split.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 10 >> gpurun_out/s3_split.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py D --reps 10 --persp 512 --stride 8 >> gpurun_out/s3_split.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 6 >> gpurun_out/s3_split.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s3_split.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['persp'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
