# round 2: warp tile shape (8x4 default vs 4x8, 16x2, 32x1) on the current kernel
set -x
for lib in libnbt.so variants/libnbt_tw4.so variants/libnbt_tw16.so variants/libnbt_tw32.so; do
  echo "== $lib" >> gpurun_out/tv13.log
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py B D >> gpurun_out/tv13.log 2>&1
  NBT_LIB=paper_2503_22588_b200/$lib python tools/trace_variants.py "C'" --bits 8 >> gpurun_out/tv13.log 2>&1
done
grep -E '^\{|^==' gpurun_out/tv13.log | cut -c1-100
