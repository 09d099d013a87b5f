"""Rewrite the measured numbers of profiles/r01_summary.md from a bench.py JSON line (and
optionally a config-E JSON), so an evidence refresh is one command:

    python tools/refresh_summary.py profiles/r01_bench.log [profiles/r01_config_e.json]
"""
import json
import re
import sys

ROOT_SUMMARY = "profiles/r01_summary.md"


def main():
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    s = open(ROOT_SUMMARY).read()
    a, b = s.index("## bench.py"), s.index("## North-star")
    r, e, c = d["roofline"], d["e2e"], d["cpu_baseline"]
    shares = ", ".join(f"{k} {v:.4f}" for k, v in d["kernel_share_of_step"].items())
    block = (
        "## bench.py (config B: 256^3 SYN map, 512 perspectives x 64x48 rays, + deltas + 1984 IDW queries)\n\n"
        f"* value: **{d['value']:.4g} rays/s** ({d['ms_per_step']:.3f} ms per MHP cycle, {d['steps']} timed steps, "
        "L2 flushed before each; the timed CUDA graphs carry event nodes only around k_id_trace; "
        f"{d['gpu_launches'] // d['steps']} libnbt launches per step)\n"
        f"* voxel-steps/s {d['voxel_steps_per_s']:.4g}, in-grid lookups/s {d['lookups_per_s']:.4g}\n"
        "* e2e through the public API from pinned host memory (one CUDA-graph replay of the public calls and the "
        f"copies per step, one synchronisation): **{e['value']:.4g} rays/s** ({e['ms_per_step']:.3f} ms per cycle; "
        f"{e['h2d_bytes_per_step']} B in, {e['d2h_bytes_per_step']} B out per cycle)\n"
        f"* roofline (k_id_trace, integer issue): achieved {r['achieved']:.2f} of {r['peak']:.1f} Tops/s = "
        f"**{r['frac']:.3f}**; kernel {r['kernel_avg_ms'] * 1e3:.0f} us per launch; DRAM traffic per launch (ncu, "
        f"cold L2) {r['traffic'] / 1e6:.2f} MB = the map once; the walk's own instruction mix tops out at 0.664 "
        "(`r01_dda_step_peak.log`)\n"
        f"* kernel share of the step (separate fully profiled run): {shares}\n")
    if c:
        block += (f"* CPU oracle ({c['cores']} host threads): {c['value']:.4g} rays/s -> GPU/oracle "
                  f"{d['value'] / c['value']:.0f}x ({c['sample']})\n")
    s = s[:a] + block + "\n" + s[b:]
    ns, D, F = d.get("north_star"), d.get("config_d_strong"), d.get("map_integration")
    if ns:
        s = re.sub(r"\* whole hot path per MHP cycle: \*\*[0-9.]+ ms\*\* \(target <= 100 ms, P:309\), [0-9.e+]+ rays/s",
                   f"* whole hot path per MHP cycle: **{ns['id_latency_ms']:.1f} ms** (target <= 100 ms, P:309), "
                   f"{ns['rays_per_s']:.4g} rays/s", s)
    if D:
        s = re.sub(r"\* one ID on one B200: \*\*[0-9.]+ ms\*\*, [0-9.e+]+ rays/s, [0-9.e+]+ lookups/s",
                   f"* one ID on one B200: **{D['id_ms']:.1f} ms**, {D['rays_per_s']:.4g} rays/s, "
                   f"{D['lookups_per_s']:.4g} lookups/s", s)
    if F:
        s = re.sub(r"\* \*\*[0-9.]+ ms per frame\*\* on the device \(~[0-9]+ points -> ~[0-9]+ filtered rays -> ~[0-9]+ "
                   r"voxel updates\), [0-9.e+]+ points/s; end to end from host numpy points [0-9.]+ ms per frame",
                   f"* **{F['ms_per_frame']:.3f} ms per frame** on the device (~{F['mean_points']:.0f} points -> "
                   f"~{F['mean_rays']:.0f} filtered rays -> ~{F['mean_voxels_updated']:.0f} voxel updates), "
                   f"{F['points_per_s']:.4g} points/s; end to end from host numpy points "
                   f"{F['e2e_ms_per_frame_p50']:.2f} ms per frame", s)
    s = re.sub(r"clocks sampled through NVML every 5 ms inside the timed region: [0-9]+ samples",
               f"clocks sampled through NVML every 5 ms inside the timed region: {d['clocks']['samples']} samples", s)
    if len(sys.argv) > 2:
        E = json.load(open(sys.argv[2]))
        s = re.sub(r"\* `r01_config_e.json`: device time per cycle p50 [0-9.]+ ms, p99 [0-9.]+ ms; wall p50 [0-9.]+ ms, "
                   r"p99 [0-9.]+ ms",
                   f"* `r01_config_e.json`: device time per cycle p50 {E['device_ms_p50']:.2f} ms, p99 "
                   f"{E['device_ms_p99']:.2f} ms; wall p50 {E['wall_ms_p50']:.2f} ms, p99 {E['wall_ms_p99']:.2f} ms", s)
    open(ROOT_SUMMARY, "w").write(s)


if __name__ == "__main__":
    main()
