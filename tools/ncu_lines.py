#!/usr/bin/env python3
"""Executed warp-instructions and stall samples per CUDA source line (from an
ncu report captured with -lineinfo + --import-source).  Usage:
ncu_lines.py report.ncu-rep kernel-regex [top]"""
import collections, csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
path, hdr = None, None
agg = collections.defaultdict(lambda: [0, 0, 0.0, ""])
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]; continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r; ie = hdr.index("Instructions Executed"); iss = hdr.index("Warp Stall Sampling (All Samples)")
        ith = hdr.index("Avg. Threads Executed"); continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:
        cur = (path, r[0], r[1])
    if not r[3] or cur is None:  # no sass on this row
        continue
    try:
        n = int(r[ie] or 0); ss = int(r[iss] or 0); th = float(r[ith] or 0)
    except ValueError:
        continue
    a = agg[cur[:2]]; a[0] += n; a[1] += ss; a[2] += n * th; a[3] = cur[2]
tot = sum(v[0] for v in agg.values()) or 1
tss = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instr {tot}  stall samples {tss}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    th = v[2] / v[0] if v[0] else 0
    print(f"{100*v[0]/tot:5.1f}% inst {100*v[1]/tss:5.1f}% stall {th:5.1f}thr  {k[0][:12]}:{k[1]:<5s} {v[3].strip()[:70]}")
