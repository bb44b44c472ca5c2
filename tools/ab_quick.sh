#!/bin/bash
# quick step-time check of the persistent-kernel configs: 10k (config [0]), 1M (config [1]), a 1.28M part
out=${1:-gpurun_out/r02_ab_quick.txt}
: > $out
one() {  # label cfg steps env...
  local lab=$1 cfg=$2 k=$3; shift 3
  env "$@" python bench.py --config $cfg --steps $k --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', '$lab', round(d['ms_per_step']*1e3,3), 'us/step', d['clocks']['sm_mhz'])" >> $out
}
for rep in 1 2; do
  one head circular_dam_break 3000
  one head three_mounds_friction 300 SWE_PERSISTENT=1
done
echo "parts8 $(SWE_PERSISTENT=1 timeout 300 python tools/run_timing.py --config channel --parts 8 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["us_per_step"],2), "us/step")')" >> $out
