"""Per source line shared-memory wavefronts (actual vs ideal) from an ncu source export.
usage: python scripts/ncu_smem.py report.ncu-rep kernel_regex [topN]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
fname, hdr, res = "?", None, {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {}
        for i, k in enumerate(r):
            hdr.setdefault(k, i)
        continue
    if hdr is None or not r[0].isdigit():
        continue
    try:
        wf = int(r[hdr["L1 Wavefronts Shared"]] or 0)
        ideal = int(r[hdr["L1 Wavefronts Shared Ideal"]] or 0)
    except (ValueError, KeyError):
        continue
    e = res.setdefault(f"{fname}:{r[0]}", [0, 0, r[1].strip()[:80]])
    e[0] += wf
    e[1] += ideal
tw = sum(v[0] for v in res.values()) or 1
ti = sum(v[1] for v in res.values())
print(f"shared wavefronts {tw}  ideal {ti}  excess {tw - ti}")
for k, (w, i, src) in sorted(res.items(), key=lambda kv: -(kv[1][0] - kv[1][1]))[:top]:
    print(f"{w:9d} ideal {i:9d} excess {w - i:9d}  {k:22s} {src}")
