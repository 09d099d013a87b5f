# refresh profiles/ from a measurement pass's gpurun_out/<tag>_* files (bench line, ncu captures, launch list)
tag=$1
python tools/refresh_traffic.py gpurun_out/$tag > /dev/null
for c in d cp8 b; do
  python tools/ncu_summary.py gpurun_out/${tag}_trace_$c.ncu-rep profiles/r02_${tag}_trace_${c}_ncu.md > /dev/null 2>&1
  python tools/sass_blocks.py gpurun_out/${tag}_trace_$c.ncu-rep --top 14 > profiles/r02_${tag}_trace_${c}_blocks.md 2>&1
done
python tools/ncu_summary.py gpurun_out/${tag}_idw.ncu-rep profiles/r02_${tag}_idw_ncu.md > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${tag}_launches.csv > profiles/r02_${tag}_launches_bench_cmd_summary.md 2>&1
cp gpurun_out/${tag}_launches.csv profiles/r02_${tag}_launches_bench_cmd.csv
cp gpurun_out/${tag}_bench.json profiles/r02_${tag}_bench.json
cp gpurun_out/${tag}_bench_s6.json profiles/r02_${tag}_bench_d_s6_world1.json
cp gpurun_out/${tag}_bench_w2.json profiles/r02_${tag}_bench_d_s6_world2_gloo.json
