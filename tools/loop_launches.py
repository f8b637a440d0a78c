"""Per-kernel mean time and DRAM bytes from an ncu --csv launch list (gpu__time_duration.sum,
dram__bytes_read.sum): python tools/loop_launches.py gpurun_out/x.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
t, b = collections.defaultdict(list), collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    k = r[ix["Kernel Name"]][:50]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    (t if r[ix["Metric Name"]] == "gpu__time_duration.sum" else b)[k].append(v)
for k in t:
    mt = sum(t[k]) / len(t[k])
    mb = sum(b[k]) / max(1, len(b[k]))
    print(f"{k:50s} n={len(t[k]):3d} mean={mt / 1e3:8.1f}us  dram={mb / 1e6:8.1f}MB  {mb / mt / 1e3:6.2f} TB/s")
