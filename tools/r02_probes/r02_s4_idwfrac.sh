# round 2 session 4: IDW per-tile sums as fractions over one denominator (NBT_IDW_FRAC=1, no reciprocal per pair) -- A/B + IDW parity tests on the variant
set -x
NBT_LIB=paper_2503_22588_b200/variants/libnbt_idwfrac.so timeout 600 python -m pytest tests -m gpu -q -k "idw or info_cost" > gpurun_out/s4_idwfrac_tests.log 2>&1; tail -2 gpurun_out/s4_idwfrac_tests.log
for i in 1 2 3; do
for lib in libnbt.so variants/libnbt_idwfrac.so; do
  echo "== $lib" >> gpurun_out/s4_idwfrac.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/idw_probe.py >> gpurun_out/s4_idwfrac.log 2>&1
done; done
cat gpurun_out/s4_idwfrac.log
