# round 2: trace register budgets (5 / 6 resident blocks of 8 warps) vs default, 2-bit and byte stores
set -x
for lib in libnbt.so variants/libnbt_mb5.so variants/libnbt_mb6.so; do
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B "C'" D >> gpurun_out/tv12.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 >> gpurun_out/tv12.log 2>&1
done
grep '^{' gpurun_out/tv12.log | cut -c1-100
