"""Summarise an ncu report (.ncu-rep) into the per-kernel numbers DESIGN.md cites.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--samples N] > profiles/x.txt

--samples: samples processed by each dvr_* launch in the report, to print
per-sample instruction and wavefront counts.
"""

from __future__ import annotations

import argparse
import csv
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1/TEX throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "global load requests"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "global load sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_red.sum", "global red requests"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--samples", type=float, default=0.0)
    args = ap.parse_args()
    out = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        print(f"== {r[head.index('Kernel Name')][:90]}")
        vals = {}
        for key, label in METRICS:
            if key in head:
                i = head.index(key)
                vals[key] = r[i]
                print(f"   {label:26s} {r[i]:>22s} {units[i]}")
        if args.samples and "smsp__inst_executed.sum" in vals:
            try:
                warp_samples = args.samples / 32.0
                inst = float(vals["smsp__inst_executed.sum"].replace(",", ""))
                print(f"   {'warp-inst / warp-sample':26s} {inst / warp_samples:22.1f}")
            except ValueError:
                pass


if __name__ == "__main__":
    main()
