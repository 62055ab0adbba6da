"""Top SASS instructions by warp-stall samples for one kernel of an ncu report.

    python tools/ncu_hot.py <report.ncu-rep> <name-substring> [top]

The source page lists one table per profiled kernel; the first kernel whose
demangled name contains <name-substring> is summarised.
"""
import csv
import io
import subprocess
import sys

rep, key = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, name, cur = [], None, []
for line in out.splitlines():
    if line.startswith('"Kernel Name"'):
        if name is not None:
            blocks.append((name, cur))
        name, cur = line, []
    elif name is not None:
        cur.append(line)
if name is not None:
    blocks.append((name, cur))
name, lines = next((n, b) for n, b in blocks if key in n)
rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
col = "Warp Stall Sampling (All Samples)"
tot = sum(int(r[col] or 0) for r in rows)
print(name[:160])
print(f"total stall samples {tot}")
addr0 = int(rows[0]["Address"], 16)
for r in sorted(rows, key=lambda r: -int(r[col] or 0))[:top]:
    n = int(r[col] or 0)
    print(f'{int(r["Address"], 16) - addr0:06x} {n:8d} {100 * n / tot:5.1f}%  {r["Source"].strip()}')
