"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of bench.py: per-kernel
counts and times over the whole run, and the kernel shares of the headline step (the launches
between the headline's first timed and last share-run k_id_trace, by launch order).

    python tools/launch_summary.py gpurun_out/final_launches.csv [--skip-trace 5 --trace 40] > profiles/x.md
"""
import collections
import csv
import re
import sys


def short(name):
    n = re.sub(r"\(.*", "", name)
    n = n.replace("nbt::<unnamed>::", "").replace("void ", "").replace("(anonymous namespace)::", "")
    return n.split("<")[0] if "k_id_trace" not in n else "k_id_trace"


def main():
    path = sys.argv[1]
    skip = int(sys.argv[sys.argv.index("--skip-trace") + 1]) if "--skip-trace" in sys.argv else 5
    take = int(sys.argv[sys.argv.index("--trace") + 1]) if "--trace" in sys.argv else 40
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        rows.append((int(r["ID"]), short(r["Kernel Name"]), float(r["Metric Value"]) / 1e3))  # us
    tot = collections.defaultdict(lambda: [0, 0.0])
    for _, k, us in rows:
        tot[k][0] += 1
        tot[k][1] += us
    print(f"# ncu launch list: {path} ({len(rows)} launches, gpu__time_duration.sum, clock control none)\n")
    print("| kernel | launches | total us | mean us |\n|---|---|---|---|")
    for k, (n, us) in sorted(tot.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {n} | {us:.1f} | {us / n:.2f} |")
    idx = [i for i, (_, k, _) in enumerate(rows) if k == "k_id_trace"]
    if len(idx) > skip:
        a = idx[skip]
        b = idx[min(len(idx) - 1, skip + take - 1)]
        # the step's other kernels follow its trace launch: extend to the next trace launch
        nxt = [i for i in idx if i > b]
        e = nxt[0] if nxt else len(rows)
        seg = rows[a:e]
        # drop launches of other blocks that started before the next trace launch
        share = collections.defaultdict(float)
        for _, k, us in seg:
            share[k] += us
        s = sum(share.values())
        n_steps = min(len(idx) - skip, take)
        print(f"\n## Kernel shares of the headline step ({n_steps} steps: trace launches #{skip}..#{skip + n_steps - 1})\n")
        print("| kernel | share | us per step |\n|---|---|---|")
        for k, us in sorted(share.items(), key=lambda x: -x[1]):
            print(f"| {k} | {us / s:.4f} | {us / n_steps:.1f} |")


if __name__ == "__main__":
    main()
