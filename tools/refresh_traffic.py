"""Write profiles/ncu_traffic_{D,C',B}.json (per-launch DRAM / L2 bytes, L1 data-pipe and issue
utilisation of k_id_trace, read by bench.py's roofline block) from one `ncu --set full` capture
per config, e.g. the ones tools/r02_probes/r02_s3_final*.sh writes.

    python tools/refresh_traffic.py gpurun_out/s3h   # reads s3h_trace_{d,cp8,b}.ncu-rep
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "msecond": 1, "usecond": 1e-3, "us": 1e-3,
         "nsecond": 1e-6, "ns": 1e-6, "ms": 1}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return dict(zip(r[0], r[1])), dict(zip(r[0], r[2]))


def main():
    prefix = sys.argv[1]
    tag = os.path.basename(prefix)
    for n, cfg, store in (("d", "D", "2-bit"), ("cp8", "C'", "8-bit"), ("b", "B", "2-bit")):
        units, m = raw(f"{prefix}_trace_{n}.ncu-rep")
        f = lambda k: float(m[k].replace(",", ""))
        u = lambda k: SCALE.get(units.get(k, ""), 1)
        req = f("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum")
        d = {"kernel": "k_id_trace", "config": cfg, "store": store,
             "dram_bytes_per_launch": f("dram__bytes_read.sum") * u("dram__bytes_read.sum")
             + f("dram__bytes_write.sum") * u("dram__bytes_write.sum"),
             "l2_bytes_per_launch": f("lts__t_sectors_srcunit_tex_op_read.sum") * 32,
             "l1_hit_rate_pct": f("l1tex__t_sector_hit_rate.pct"),
             "duration_ms": f("gpu__time_duration.sum") * u("gpu__time_duration.sum"),
             "source": f"ncu --set full --clock-control none, one launch ({tag}_trace_{n}.ncu-rep; "
                       f"profiles/r02_{tag}_trace_{n}_ncu.md): dram__bytes_read.sum + dram__bytes_write.sum; "
                       f"L2 = lts__t_sectors_srcunit_tex_op_read.sum x 32 B",
             "l1_data_pipe_wavefronts_pct": f("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
             "l1_wavefronts_per_request": f("l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum") / req,
             "l1_sectors_per_request": f("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum") / req,
             "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
             "alu_pipe_pct": f("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
             "fma_pipe_pct": f("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
             "source_l1": "same capture: l1tex__data_pipe_lsu_wavefronts (pct of peak, elapsed), "
                          "t_output_wavefronts / t_requests, t_sectors / t_requests (global loads); smsp__issue_active"}
        with open(os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg}.json"), "w") as fh:
            json.dump(d, fh, indent=1)
        print(cfg, {k: (round(v, 3) if isinstance(v, float) else v) for k, v in d.items() if not k.startswith("source")})


if __name__ == "__main__":
    main()
