"""Top SASS instructions by warp-stall samples for one kernel of an ncu report.

    python tools/ncu_hot.py <report.ncu-rep> <kernel-regex> [top]
Prints the hottest instructions (stall samples, share) and, for the hottest
loop, the per-instruction listing with samples, so latency chains are visible.
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
print(f"total stall samples {tot}")
hot = sorted(rows, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:top]
addr0 = int(rows[0]["Address"], 16)
for r in hot:
    n = int(r["Warp Stall Sampling (All Samples)"] or 0)
    print(f'{int(r["Address"], 16) - addr0:06x} {n:8d} {100 * n / tot:5.1f}%  {r["Source"].strip()}')
