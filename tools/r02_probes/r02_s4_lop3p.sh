# round 2 session 4: "x first" from one LOP3 with a predicate output instead of two compares (12 instead of 13 per step) -- A/B, GPU suite, 1500-seed fuzz
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s4_lop3p_tests.log 2>&1; tail -2 gpurun_out/s4_lop3p_tests.log
NBT_FUZZ_SEEDS=1500 timeout 1500 python -m pytest tests -m gpu -k fuzz -q > gpurun_out/s4_lop3p_fuzz1500.log 2>&1; tail -2 gpurun_out/s4_lop3p_fuzz1500.log
for i in 1 2; do
for lib in variants/libnbt_pred2.so libnbt.so; do
  echo "== $lib" >> gpurun_out/s4_lop3p.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 8 >> gpurun_out/s4_lop3p.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 5 >> gpurun_out/s4_lop3p.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s4_lop3p.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['persp'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
