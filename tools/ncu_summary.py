#!/usr/bin/env python3
"""Summarise an ncu report: key raw metrics per kernel + top SASS stall lines.
Usage: ncu_summary.py report.ncu-rep [kernel-regex]"""
import csv, io, subprocess, sys, collections

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else None
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if kre and kre not in name:
        continue
    print("==", name[:70])
    for w in WANT:
        if w in hdr:
            i = hdr.index(w)
            print(f"   {w:58s} {r[i]} {units[i]}")
# stall reasons
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
drows = list(csv.reader(io.StringIO(det)))
h = drows[0]
ki, si, mi, vi = h.index("Kernel Name"), h.index("Section Name"), h.index("Metric Name"), h.index("Metric Value")
for r in drows[1:]:
    if kre and kre not in r[ki]:
        continue
    if r[si] in ("Warp State Statistics", "Scheduler Statistics") or "Stall" in r[mi]:
        print(f"   [{r[ki][:18]}] {r[mi][:55]:55s} {r[vi]}")
