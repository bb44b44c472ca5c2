#!/bin/bash
# the linked exchange's cost per step at a part's size (channel scaled to ~1.28M / ~2.56M cells):
# unlinked vs self-linked, graph loop vs persistent kernel
out=${OUT:-gpurun_out/r02_ab_link.txt}
: > $out
for sc in ${SCALES:-0.125 0.25}; do
  for P in 0 1; do
    for L in "" "--self-link"; do
      r=$(SWE_PERSISTENT=$P timeout 300 python tools/run_timing.py --config channel --scale $sc --steps 400 $L 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["us_per_step"],2), "us/step", d["info"]["tiles"], "tiles")')
      echo "scale$sc persistent=$P ${L:-unlinked} $r" >> $out
    done
  done
done
