# round 2 session 4: byte store packed bottom-up (one funnel shift right per visit on the ALU pipe instead of an FMA-pipe IMAD) -- A/B on C' + GPU suite + 2000-seed fuzz
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s4_revpack_tests.log 2>&1; tail -2 gpurun_out/s4_revpack_tests.log
NBT_FUZZ_SEEDS=2000 timeout 1500 python -m pytest tests -m gpu -k fuzz -q > gpurun_out/s4_revpack_fuzz.log 2>&1; tail -2 gpurun_out/s4_revpack_fuzz.log
for i in 1 2 3; do
for lib in variants/libnbt_fwdpack.so libnbt.so; do
  echo "== $lib" >> gpurun_out/s4_revpack.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" B --bits 8 --reps 5 >> gpurun_out/s4_revpack.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s4_revpack.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['persp'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
