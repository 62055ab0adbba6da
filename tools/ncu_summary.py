"""Summarise an ncu report (.ncu-rep) into the per-kernel numbers DESIGN.md cites.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--samples N] > profiles/x.txt
    python tools/ncu_summary.py rep --samples N --kernel dvr_adjoint \
        --json-out profiles/ncu_r02.json --key C4/fused_tape [--file profiles/x.txt]

The report may also be the raw page saved as CSV (`ncu -i rep --page raw --csv > x.csv`).
--samples: samples processed by each dvr_* launch in the report, to print
per-sample instruction and wavefront counts.  --json-out/--key: merge the
numbers of the first launch whose name contains --kernel into the JSON file
bench.py reads for its roofline (achieved = these DRAM bytes / live launch time).
"""

from __future__ import annotations

import json
import os

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
    ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 red sectors"),
    ("lts__t_sectors_srcunit_tex_op_red.sum.pct_of_peak_sustained_elapsed", "L2 red sectors % peak"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--samples", type=float, default=0.0)
    ap.add_argument("--json-out")
    ap.add_argument("--key")
    ap.add_argument("--kernel", default="dvr_")
    ap.add_argument("--file", default="", help="the summary file this entry is cited from")
    ap.add_argument("--state", default="bench.py fixed dense state (iteration 1)")
    args = ap.parse_args()
    if args.report.endswith(".csv"):   # a saved `ncu -i rep --page raw --csv` page
        with open(args.report) as f:
            out = f.read()
    else:
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
        if args.json_out and args.key and args.kernel in r[head.index("Kernel Name")]:
            _merge_json(args, vals, units, head, r)
            args.json_out = None
        if args.samples and "smsp__inst_executed.sum" in vals:
            try:
                warp_samples = args.samples / 32.0
                inst = float(vals["smsp__inst_executed.sum"].replace(",", ""))
                print(f"   {'warp-inst / warp-sample':26s} {inst / warp_samples:22.1f}")
            except ValueError:
                pass


def _num(v):
    return float(str(v).replace(",", ""))


def _merge_json(args, vals, units, head, row):
    """One launch's numbers, normalised to bytes / ms / per-sample, into --json-out."""
    def unit_scale(key):
        u = units[head.index(key)]
        return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                "nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0,
                "ms": 1.0, "second": 1e3, "s": 1e3}.get(u, 1.0)
    g = lambda k: _num(vals[k]) * unit_scale(k)  # noqa: E731
    dur_ms = g("gpu__time_duration.sum")
    e = {"kernel": row[head.index("Kernel Name")][:120], "state": args.state,
         "file": args.file, "duration_ms": dur_ms,
         "dram_bytes": g("dram__bytes_read.sum") + g("dram__bytes_write.sum"),
         "issue_active_pct": _num(vals["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
         "l1tex_pct": _num(vals["l1tex__throughput.avg.pct_of_peak_sustained_elapsed"]),
         "l2_pct": _num(vals["lts__throughput.avg.pct_of_peak_sustained_elapsed"]),
         "dram_pct": _num(vals["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]),
         "occupancy_pct": _num(vals["sm__warps_active.avg.pct_of_peak_sustained_active"]),
         "registers": _num(vals["launch__registers_per_thread"])}
    red = _num(vals.get("l1tex__t_requests_pipe_lsu_mem_global_op_red.sum", 0))
    e["red_requests"] = red
    e["red_requests_per_s"] = red / (dur_ms / 1e3) if dur_ms else None
    if "lts__t_sectors_srcunit_tex_op_red.sum" in vals:   # 32-byte sectors the L2 reduced
        e["red_sectors"] = _num(vals["lts__t_sectors_srcunit_tex_op_red.sum"])
        e["red_sectors_pct_of_l2_peak"] = _num(
            vals["lts__t_sectors_srcunit_tex_op_red.sum.pct_of_peak_sustained_elapsed"])
    if args.samples:
        e["samples"] = args.samples
        e["warp_inst_per_sample"] = _num(vals["smsp__inst_executed.sum"]) / (args.samples / 32)
        e["gather_requests_per_sample"] = _num(
            vals["l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"]) / (args.samples / 32)
        e["dram_bytes_per_sample"] = e["dram_bytes"] / args.samples
    d = {}
    if os.path.exists(args.json_out):
        with open(args.json_out) as f:
            d = json.load(f)
    d[args.key] = e
    with open(args.json_out, "w") as f:
        json.dump(d, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
