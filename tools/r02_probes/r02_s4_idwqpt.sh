# round 2 session 4: IDW queries per thread 3 / 4 / 5 (QPT 5: 126 registers, 250 blocks = one wave of 2 per SM) -- A/B + IDW parity on QPT 5
set -x
NBT_LIB=paper_2503_22588_b200/variants/libnbt_qpt5.so timeout 600 python -m pytest tests -m gpu -q -k "idw or info_cost" > gpurun_out/s4_idwqpt_tests.log 2>&1; tail -2 gpurun_out/s4_idwqpt_tests.log
for i in 1 2 3; do
for lib in libnbt.so variants/libnbt_qpt4.so variants/libnbt_qpt5.so; do
  echo "== $lib" >> gpurun_out/s4_idwqpt.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/idw_probe.py >> gpurun_out/s4_idwqpt.log 2>&1
done; done
cat gpurun_out/s4_idwqpt.log | grep -v "^==" | python -c "
import sys,json,collections
d=collections.defaultdict(list)
for l in sys.stdin:
    try: r=json.loads(l); d[(r['lib'],r['n_persp'])].append(r['us_p50'])
    except Exception: pass
for k,v in sorted(d.items()): print(k, [round(x,2) for x in v])
"
