# round 2 session 4: 2-bit word address on the ALU pipe as the default (GPU suite + 2000-seed fuzz); A/B against the IMAD.WIDE address and the one-LOP3 x-first predicate on top
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s4_addrlea_tests.log 2>&1; tail -2 gpurun_out/s4_addrlea_tests.log
NBT_FUZZ_SEEDS=2000 timeout 1500 python -m pytest tests -m gpu -k fuzz -q > gpurun_out/s4_addrlea_fuzz.log 2>&1; tail -2 gpurun_out/s4_addrlea_fuzz.log
for i in 1 2; do
for lib in variants/libnbt_wide.so libnbt.so variants/libnbt_pred3.so; do
  echo "== $lib" >> gpurun_out/s4_addrlea.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 8 >> gpurun_out/s4_addrlea.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 5 >> gpurun_out/s4_addrlea.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --reps 4 >> gpurun_out/s4_addrlea.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s4_addrlea.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['persp'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
