"""Summarise ncu captures (run under gpurun) into profiles/<tag>_summary.md and
profiles/traffic.json (per-launch DRAM traffic of each kernel, read by bench.py).

usage: python scripts/summarize_profiles.py <tag> <launches.csv> <full.ncu-rep>
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PX = 8192 * 8192


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) < len(h) or (mi is not None and r[mi] != "gpu__time_duration.sum"):
            continue
        agg.setdefault(r[ki], []).append(float(r[vi].replace(",", "")) / 1e3)  # ns -> us
    return agg


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        un = dict(zip(h, u))
        res.append((d, un))
    return res


def short(name):
    for k in ("k_local_wf", "k_local", "k_seams", "k_resolve", "k_final"):
        if k in name:
            return k
    return name.split("(")[0][-50:]


def mbytes(v, unit):
    v = float(v.replace(",", ""))
    return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)


def main():
    tag, lcsv, rep = sys.argv[1], sys.argv[2], sys.argv[3]
    L = launches(lcsv)
    R = raw(rep)
    lines = [f"# ncu summary — {tag}", "",
             "Workload: 8192x8192 random binary d=0.5 (bench.py), 1x B200. Launch times from "
             "`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised: compare "
             "shares, not absolutes); traffic/occupancy from one `ncu --set full` capture per kernel.", "",
             "## Launch list (our kernels, mean per launch)", "", "| kernel | launches | mean us | share of step |",
             "|---|---|---|---|"]
    ours = {short(k): v for k, v in L.items() if short(k).startswith("k_")}
    tot = sum(sum(v) / len(v) for v in ours.values())
    for k, v in ours.items():
        m = sum(v) / len(v)
        lines.append(f"| {k} | {len(v)} | {m:.1f} | {100 * m / tot:.0f}% |")
    lines += ["", f"Sum of our kernels per step: {tot:.1f} us.", "", "## Full-set metrics (one launch each)", "",
              "| kernel | dur us | DRAM read MB | DRAM write MB | B/px | DRAM GB/s | achieved occ. | IPC | "
              "regs | smem/CTA |", "|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for d, un in R:
        k = short(d["Kernel Name"])
        if k not in ("k_local_wf", "k_local", "k_seams", "k_resolve", "k_final"):
            continue
        dur = float(d["gpu__time_duration.sum"].replace(",", ""))
        if un["gpu__time_duration.sum"] == "ms":
            dur *= 1e3
        rd = mbytes(d["dram__bytes_read.sum"], un["dram__bytes_read.sum"])
        wr = mbytes(d["dram__bytes_write.sum"], un["dram__bytes_write.sum"])
        occ = d.get("sm__warps_active.avg.pct_of_peak_sustained_active", "")
        ipc = d.get("sm__inst_executed.avg.per_cycle_active", "")
        regs = d.get("launch__registers_per_thread", "")
        smem = d.get("launch__shared_mem_per_block_dynamic", "")
        lines.append(f"| {k} | {dur:.1f} | {rd:.1f} | {wr:.1f} | {(rd + wr) * 1e6 / PX:.2f} | "
                     f"{(rd + wr) * 1e6 / (dur * 1e-6) / 1e9:.0f} | {occ} | {ipc} | {regs} | {smem} |")
        key = {"k_local_wf": "local_ms", "k_local": "local_ms", "k_seams": "merge_ms", "k_resolve": "final_ms", "k_final": "final_ms"}[k]
        traffic[key] = traffic.get(key, 0.0) + (rd + wr) * 1e6  # final_ms spans (d2) resolve + (e)
    os.makedirs(os.path.join(REPO, "profiles"), exist_ok=True)
    with open(os.path.join(REPO, "profiles", f"{tag}_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(os.path.join(REPO, "profiles", "traffic.json"), "w") as f:
        json.dump({**traffic, "source": f"profiles/{tag}_summary.md", "unit": "bytes per launch"}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
