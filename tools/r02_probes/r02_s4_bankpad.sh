# round 2 session 4: L1-bank padding of the linear store (rows an odd number of words, planes 17 words mod 32) -- A/B on B / D / C' + parity tests on the variant
set -x
NBT_LIB=paper_2503_22588_b200/variants/libnbt_bankpad.so timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s4_bankpad_tests.log 2>&1; tail -2 gpurun_out/s4_bankpad_tests.log
for i in 1 2; do
for lib in libnbt.so variants/libnbt_bankpad.so; do
  echo "== $lib" >> gpurun_out/s4_bankpad.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 8 >> gpurun_out/s4_bankpad.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 5 >> gpurun_out/s4_bankpad.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s4_bankpad.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['persp'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
NBT_LIB=paper_2503_22588_b200/variants/libnbt_bankpad.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/s4_bankpad_d python tools/trace_variants.py D --reps 1 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep | tail -2
