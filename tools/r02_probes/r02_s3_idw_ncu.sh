# round 2 session 3: ncu --set full of the IDW kernels (warp-per-unit k_idw_pairs vs block-per-entry k_idw_entry), 512 perspectives
set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_idw -s 3 -c 1 -o gpurun_out/s3_idw_pairs python tools/idw_probe.py > /dev/null 2>&1
NBT_LIB=paper_2503_22588_b200/variants/libnbt_idw_entry.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_idw -s 3 -c 1 -o gpurun_out/s3_idw_entry python tools/idw_probe.py > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
