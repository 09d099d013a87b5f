# round 2 session 4: bank padding as the default (GPU suite + 1500-seed fuzz) and the 2-bit word address on the ALU pipe (SHF + LEA + LEA.HI.X) -- A/B
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s4_bankpad2_tests.log 2>&1; tail -2 gpurun_out/s4_bankpad2_tests.log
NBT_FUZZ_SEEDS=1500 timeout 1500 python -m pytest tests -m gpu -k fuzz -q > gpurun_out/s4_bankpad2_fuzz.log 2>&1; tail -2 gpurun_out/s4_bankpad2_fuzz.log
for i in 1 2; do
for lib in variants/libnbt_nopad.so libnbt.so variants/libnbt_addrlea.so; do
  echo "== $lib" >> gpurun_out/s4_bankpad2.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D --reps 8 >> gpurun_out/s4_bankpad2.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 --reps 5 >> gpurun_out/s4_bankpad2.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s4_bankpad2.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['persp'], d['store'], round(d['trace_ms'],4), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
NBT_LIB=paper_2503_22588_b200/variants/libnbt_addrlea.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_id_trace -c 1 -o gpurun_out/s4_addrlea_d python tools/trace_variants.py D --reps 1 > /dev/null 2>&1
