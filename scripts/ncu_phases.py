"""Instruction counts of kernel (a) per source-line range (phases), from an ncu source export.
usage: python scripts/ncu_phases.py report.ncu-rep kernel_regex file.cu start1:name1 start2:name2 ..."""
import csv, io, subprocess, sys
rep, kre, fname = sys.argv[1], sys.argv[2], sys.argv[3]
marks = sorted((int(a.split(":")[0]), a.split(":")[1]) for a in sys.argv[4:])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
cur, hdr = "?", None
acc = {}
other = {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {}
        for i, k in enumerate(r):
            hdr.setdefault(k, i)
        continue
    if hdr is None or not r[0].isdigit():
        continue
    try:
        inst = int(r[hdr["Instructions Executed"]])
        samp = int(r[hdr["Warp Stall Sampling (All Samples)"]])
    except (ValueError, KeyError):
        continue
    ln = int(r[0])
    if cur != fname:
        other[cur] = other.get(cur, 0) + inst
        continue
    name = "pre"
    for s, n in marks:
        if ln >= s:
            name = n
    a = acc.setdefault(name, [0, 0])
    a[0] += inst
    a[1] += samp
tot = sum(v[0] for v in acc.values()) + sum(other.values())
ts = sum(v[1] for v in acc.values()) or 1
print(f"total instructions {tot/1e6:.1f} M")
for s, n in [(0, "pre")] + marks:
    if n in acc:
        print(f"  {n:14s} {acc[n][0]/1e6:8.2f} M inst  {100*acc[n][0]/tot:5.1f}%   samples {100*acc[n][1]/ts:5.1f}%")
for k, v in other.items():
    print(f"  [{k}] {v/1e6:8.2f} M inst (inlined helpers)")
