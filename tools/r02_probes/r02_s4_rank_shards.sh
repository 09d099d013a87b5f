# round 2 session 4: the strided rank shards of config D (N = 2 / 4 / 8) traced one at a time on one GPU, final build -- per-shard trace time against the full launch
set -x
NBT_LIB= python tools/trace_variants.py D --reps 5 > gpurun_out/s4c_rank_shards.log 2>&1
for n in 2 4 8; do
  for k in $(seq 0 $((n-1))); do
    python tools/trace_variants.py D --reps 5 --persp $((4096/n)) --stride $n --offset $k >> gpurun_out/s4c_rank_shards.log 2>&1
  done
done
python - <<'PY'
import json
rows=[json.loads(l) for l in open('gpurun_out/s4c_rank_shards.log') if l.startswith('{')]
full=rows[0]['trace_ms']; print('full', round(full,4))
i=1
for n in (2,4,8):
    sh=rows[i:i+n]; i+=n
    t=[r['trace_ms'] for r in sh]
    print(n, 'max', round(max(t),4), 'mean', round(sum(t)/n,4), 'linear', round(full/n,4), 'eff', round(full/n/max(t),4), 'max/mean', round(max(t)/(sum(t)/n),4))
PY
