"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel.

    python tools/launch_summary.py profiles/r01_launches.csv > profiles/r01_launches_summary.txt
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr, rows = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    name = r[ki].split("(")[0][:80]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * SCALE[r[ui]]
tot = sum(t for _, t in agg.values())
print("ncu --metrics gpu__time_duration.sum --clock-control none -c 400 "
      "python bench.py --steps 2 --warmup 3 --no-cpu-baseline")
print("(cold-cache, serialised launches: compare shares with the bench's CUDA-event times)\n")
for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:10.3f} ms {100 * t / tot:6.2f}%  x{n:3d}  {name}")
