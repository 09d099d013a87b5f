# round 2 session 4: f1 (per-voxel-probability store) with byte loads through PTX -- A/B on B / C' / D (prob) + the GPU suite
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4_prob_tests.log 2>&1; tail -2 gpurun_out/s4_prob_tests.log
for i in 1 2; do
for lib in variants/libnbt_byteldg.so libnbt.so; do
  echo "== $lib" >> gpurun_out/s4_prob.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B "C'" D --prob --reps 5 >> gpurun_out/s4_prob.log 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/s4_prob.log'):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l); print(' ', d['config'], d['persp'], d['store'], round(d['trace_ms'],4), round(d['rays_per_s']/1e9,3), d['checksum'])
    except Exception: print(l.rstrip()[:200])
"
