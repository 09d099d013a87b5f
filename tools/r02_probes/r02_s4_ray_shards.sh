# round 2 session 4: config D's ray split (every perspective's 32-ray units dealt over N ranks) traced one shard at a time -- balance against the strided perspective shards
set -x
python tools/trace_variants.py D --reps 5 > gpurun_out/s4_ray_shards.log 2>&1
for n in 2 4 8; do
  for k in $(seq 0 $((n-1))); do
    python tools/trace_variants.py D --reps 5 --ray-world $n --ray-rank $k >> gpurun_out/s4_ray_shards.log 2>&1
  done
done
python - <<'PY'
import json
rows=[json.loads(l) for l in open('gpurun_out/s4_ray_shards.log') if l.startswith('{')]
full=rows[0]['trace_ms']; print('full', round(full,4), rows[0]['checksum'])
i=1
for n in (2,4,8):
    sh=rows[i:i+n]; i+=n
    t=[r['trace_ms'] for r in sh]
    print(n, 'max', round(max(t),4), 'mean', round(sum(t)/n,4), 'linear', round(full/n,4), 'eff', round(full/n/max(t),4), 'max/mean', round(max(t)/(sum(t)/n),4), 'lookups sum', sum(r['lookups'] for r in sh))
PY
grep -v '^{' gpurun_out/s4_ray_shards.log | tail -3
