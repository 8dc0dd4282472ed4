"""Aggregate an ncu 'cuda,sass' source export per CUDA source line.
usage: python scripts/ncu_lines.py report.ncu-rep kernel_regex [topN]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
fname, seen, res = "?", set(), []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        if r[1] in seen and len(seen) > 0:
            pass
        seen.add(r[1])
        continue
    if r[0] == "Line No" or r[0] == "":
        continue
    try:
        samp, inst = int(r[4]), int(r[7])
    except (ValueError, IndexError):
        continue
    res.append((samp, inst, f"{fname}:{r[0]}", r[1].strip()[:100]))
tot = sum(x[0] for x in res) or 1
print("total stall samples", tot, " instructions", sum(x[1] for x in res))
for s, i, loc, src in sorted(res, reverse=True)[:top]:
    print(f"{s:7d} {100*s/tot:5.1f}%  inst {i:10d}  {loc:22s} {src}")
