#!/bin/bash
# (record of a reverted experiment: the switch it sets no longer exists; DESIGN.md §4 / §9)
# A/B of the persistent kernel's tile schedule: round robin vs dynamic (SWE_RUN_DYN=1), and the graph loop
out=gpurun_out/r02_ab_dyn.txt
: > $out
one() {  # label cfg env...
  local lab=$1 cfg=$2; shift 2
  env "$@" python bench.py --config $cfg --steps 200 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', '$lab', round(d['ms_per_step']*1e3,2), 'us/step', round(d['value']/1e9,3), 'G/s', d['clocks']['sm_mhz'], 'grid_run', d['roofline']['layout']['grid_run'])" >> $out
}
for rep in 1 2; do
  for cfg in three_mounds_friction circular_dam_break; do
    one static $cfg SWE_PERSISTENT=1 SWE_RUN_DYN=0
    one dyn $cfg SWE_PERSISTENT=1 SWE_RUN_DYN=1
  done
  for cfg in channel sloping_wet_dry; do
    one graph $cfg SWE_PERSISTENT=0
    one static $cfg SWE_PERSISTENT=1 SWE_RUN_DYN=0
    one dyn $cfg SWE_PERSISTENT=1 SWE_RUN_DYN=1
  done
done
for p in 8 4; do
  for lab in "graph SWE_PERSISTENT=0" "static SWE_PERSISTENT=1 SWE_RUN_DYN=0" "dyn SWE_PERSISTENT=1 SWE_RUN_DYN=1"; do
    set -- $lab
    l=$1; shift
    echo "parts$p $l $(env "$@" timeout 300 python tools/run_timing.py --config channel --parts $p 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["us_per_step"],2), "us/step")')" >> $out
  done
done
