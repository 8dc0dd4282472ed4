"""Summarise an ncu --csv launch log: mean time / DRAM bytes per kernel."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
acc = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[hdr + 1:]:
    name = r[ki].split("<")[0].split("(")[0].replace("void ", "").replace("cclk::", "")
    acc[name][r[mi]].append(float(r[vi].replace(",", "")))
for k, d in acc.items():
    t = d["gpu__time_duration.sum"]
    rd, wr = d.get("dram__bytes_read.sum", [0]), d.get("dram__bytes_write.sum", [0])
    print(f"{k:12s} n={len(t):3d} mean {sum(t)/len(t)/1e3:8.1f} us  read {sum(rd)/len(rd)/1e6:8.1f} MB  write {sum(wr)/len(wr)/1e6:8.1f} MB")
