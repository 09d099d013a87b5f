# round 2 session 4: byte-store loads through inline PTX (zero-extended into a 32-bit register, no re-masking before the packing) -- A/B on C' (byte store) + GPU suite
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4_byteasm_tests.log 2>&1; tail -2 gpurun_out/s4_byteasm_tests.log
for i in 1 2 3; do
for lib in variants/libnbt_byteldg.so libnbt.so; do
  echo "== $lib" >> gpurun_out/s4_byteasm.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 6 >> gpurun_out/s4_byteasm.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B --bits 8 --reps 8 >> gpurun_out/s4_byteasm.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s4_byteasm.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['persp'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
