"""Warp instructions and SIMT efficiency of kernel (a) per phase, from an
`ncu --set full --import-source on` capture: every SASS instruction is
attributed to its innermost ccl_kernels.cu line inside local_band_tiles, and
lines to phases by the `// ----` markers of the source.
usage: python scripts/ncu_phase_inst.py report.ncu-rep [tiles]"""
import collections
import csv
import io
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep = sys.argv[1]
tiles = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      "regex:k_local_band"], capture_output=True, text=True).stdout
src = open(os.path.join(REPO, "paper_1712_09789_b200", "csrc", "ccl_kernels.cu")).read().splitlines()
start = next(i for i, l in enumerate(src) if "void local_band_tiles(" in l) + 1
end = next(i for i in range(start, len(src)) if src[i].startswith("template <class C, bool TMA>") and
           "k_local_band" in src[i + 2]) + 1
marks = [(start, "prologue / tile loop head")]
for i in range(start, end):
    l = src[i - 1].strip()
    if l.startswith("// ----"):
        marks.append((i, l[7:].split(":")[0].strip()[:40]))
cur = hdr = None
seen, skip, last = set(), False, None
n_by, t_by = collections.Counter(), collections.Counter()
lines_of = collections.defaultdict(list)
ninst, tinst = {}, {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        skip = cur in seen
        seen.add(cur)
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if skip or hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        last = int(r[0])
    if not r[2]:
        continue
    try:
        ninst[r[2]] = int(r[hdr.index("Instructions Executed")] or 0)
        tinst[r[2]] = int(r[hdr.index("Thread Instructions Executed")] or 0)
    except ValueError:
        continue
    lines_of[r[2]].append((cur, last))


def phase(line):
    name = "helpers"
    for ln, nm in marks:
        if line >= ln:
            name = nm
    return name


for a, ls in lines_of.items():
    k = [l for f, l in ls if f == "ccl_kernels.cu" and start <= l <= end]
    ph = phase(k[0]) if k else "helpers (" + ls[0][0] + ")"
    n_by[ph] += ninst[a]
    t_by[ph] += tinst[a]
tot = sum(n_by.values())
print(f"kernel (a) k_local_band: {tot} warp instructions = {tot / tiles / 4:.0f} per warp per tile "
      f"({tiles} tiles, 4 warps); SIMT = thread instructions / warp instruction")
for ph, v in n_by.most_common():
    print(f"  {v / tiles / 4:7.1f} /warp/tile  {100 * v / tot:5.1f}%  SIMT {t_by[ph] / max(v, 1):5.1f}  {ph}")
