"""Aggregate an ncu source export per CUDA source line, with the dominant stall reasons.
usage: python scripts/ncu_lines.py report.ncu-rep kernel_regex [topN]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
REASONS = ["stall_barrier", "stall_branch_resolving", "stall_long_sb", "stall_short_sb", "stall_wait", "stall_mio",
           "stall_math", "stall_not_selected", "stall_selected", "stall_dispatch", "stall_lg", "stall_no_inst"]
fname, hdr, res = "?", None, {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = {}
        for i, k in enumerate(r):
            hdr.setdefault(k, i)
        continue
    if hdr is None:
        continue
    try:
        samp = int(r[hdr["Warp Stall Sampling (All Samples)"]])
        inst = int(r[hdr["Instructions Executed"]])
    except (ValueError, IndexError, KeyError):
        continue
    key = f"{fname}:{r[0]}"
    e = res.setdefault(key, [0, 0, {k: 0 for k in REASONS}, r[1].strip()[:90]])
    e[0] += samp
    e[1] += inst
    for k in REASONS:
        try:
            e[2][k] += int(r[hdr[k]])
        except (ValueError, KeyError):
            pass
tot = sum(v[0] for v in res.values()) or 1
print("total stall samples", tot, " instructions", sum(v[1] for v in res.values()))
for key, (s, i, st, src) in sorted(res.items(), key=lambda kv: -kv[1][0])[:top]:
    rs = sorted(st.items(), key=lambda kv: -kv[1])[:2]
    why = " ".join(f"{k[6:]}:{100 * v / max(s, 1):.0f}%" for k, v in rs if v)
    print(f"{s:7d} {100 * s / tot:5.1f}%  inst {i:10d}  {key:22s} {why:32s} {src}")
