"""Summarise an ncu --set full capture (one kernel launch) into markdown + JSON.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_trace_ncu.md [--traffic profiles/ncu_traffic_B.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe % of peak"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe % of peak"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe % of peak"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 data-pipe wavefronts % of peak"),
    ("sm__cycles_active.avg", "SM active cycles (mean over SMs)"),
    ("gpc__cycles_elapsed.max", "elapsed cycles"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp instr"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__t_sector_hit_rate.pct", "L1 sector hit rate %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 throughput % of peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 read sectors from L1"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit rate %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    vals = rows[2:]
    return hdr, units, vals


def main():
    rep, md = sys.argv[1], sys.argv[2]
    traffic = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    hdr, units, vals = raw(rep)
    lines = [f"# ncu --set full summary: `{rep}`", ""]
    for v in vals:
        d = dict(zip(hdr, v))
        u = dict(zip(hdr, units))
        lines.append(f"## {d.get('Kernel Name', '?')[:120]}")
        lines.append(f"grid {d.get('Grid Size', '')} block {d.get('Block Size', '')}")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for k, name in KEYS:
            if k in d:
                lines.append(f"| {name} (`{k}`) | {d[k]} {u.get(k, '')} |")
        stalls = [(k, float(d[k].replace(",", ""))) for k in hdr
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and d.get(k)]
        tot = sum(x for _, x in stalls) or 1.0
        lines.append("")
        lines.append("| stall reason (PC sampling) | share |")
        lines.append("|---|---|")
        for k, x in sorted(stalls, key=lambda t: -t[1])[:10]:
            lines.append(f"| {k.replace('smsp__pcsamp_warps_issue_stalled_', '')} | {x / tot:.3f} |")
        lines.append("")
        if traffic:
            def to_bytes(key):
                x = float(d.get(key, "0").replace(",", "") or 0)
                unit = u.get(key, "byte").lower()
                mult = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(unit, 1)
                return x * mult
            tb = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
            json.dump({"kernel": d.get("Kernel Name", "")[:200], "dram_bytes_per_launch": tb,
                       "source": rep, "note": "ncu --set full (cache control: flush all) one launch"},
                      open(traffic, "w"), indent=1)
    open(md, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
