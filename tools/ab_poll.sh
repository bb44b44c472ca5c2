#!/bin/bash
# (record of a reverted experiment: the switch it sets no longer exists; DESIGN.md §4 / §9)
# persistent kernel: longest poll back-off (SWE_POLL_CAP ns)
out=gpurun_out/r02_ab_poll.txt
: > $out
one() {  # label cfg steps env...
  local lab=$1 cfg=$2 k=$3; shift 3
  env "$@" python bench.py --config $cfg --steps $k --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', '$lab', round(d['ms_per_step']*1e3,3), 'us/step', d['clocks']['sm_mhz'])" >> $out
}
for rep in 1 2; do
  for cap in 1024 256 128 64; do
    one cap$cap circular_dam_break 3000 SWE_POLL_CAP=$cap
    one cap$cap three_mounds_friction 300 SWE_PERSISTENT=1 SWE_POLL_CAP=$cap
  done
done
for cap in 1024 256 64; do
  echo "parts8 cap$cap $(SWE_PERSISTENT=1 SWE_POLL_CAP=$cap timeout 300 python tools/run_timing.py --config channel --parts 8 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["us_per_step"],2), "us/step")')" >> $out
done
