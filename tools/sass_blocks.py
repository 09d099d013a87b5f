"""Per-basic-block instruction mix of one kernel launch from an ncu report's source page:
runs of consecutive SASS instructions with the same execution count, largest share first,
with the thread instructions per run and the stall samples.

    python tools/sass_blocks.py gpurun_out/x.ncu-rep [--top 14] [--dump START END]
"""
import csv
import io
import subprocess
import sys


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr = r[1]
    return [dict(zip(hdr, x)) for x in r[2:]]


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 14
    rs = rows(rep)
    if "--dump" in sys.argv:
        i = sys.argv.index("--dump")
        a, b = int(sys.argv[i + 1]), int(sys.argv[i + 2])
        for k, x in enumerate(rs[a:b], a):
            print(k, x["Instructions Executed"], x["Avg. Threads Executed"], x["Source"].strip())
        return
    runs = []
    cur = None
    for k, x in enumerate(rs):
        n = int(x["Instructions Executed"] or 0)
        if cur and cur["n"] == n:
            cur["instr"] += 1
            cur["thr"] += int(x["Thread Instructions Executed"] or 0)
            cur["samples"] += int(x["# Samples"] or 0)
            cur["ops"].append(x["Source"].split()[0] if x["Source"].split() else "")
        else:
            cur = {"start": k, "n": n, "instr": 1, "thr": int(x["Thread Instructions Executed"] or 0),
                   "samples": int(x["# Samples"] or 0), "ops": [x["Source"].split()[0] if x["Source"].split() else ""]}
            runs.append(cur)
    tot_w = sum(r["n"] * r["instr"] for r in runs)
    tot_t = sum(r["thr"] for r in runs)
    print(f"warp instructions {tot_w}, thread instructions {tot_t} ({tot_t / max(tot_w, 1):.2f} lanes per warp instr)")
    print("| first row | executions | instructions | share of warp instr | share of thread instr | stall samples | first opcodes |")
    print("|---|---|---|---|---|---|---|")
    for r in sorted(runs, key=lambda r: -r["n"] * r["instr"])[:top]:
        print(f"| {r['start']} | {r['n']} | {r['instr']} | {r['n'] * r['instr'] / tot_w:.3f} | {r['thr'] / tot_t:.3f} | "
              f"{r['samples']} | {' '.join(r['ops'][:6])} |")


if __name__ == "__main__":
    main()
