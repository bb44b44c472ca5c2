#!/bin/bash
# A/B of the persistent kernel's per-step acquire (fence.acq_rel.gpu: L1 invalidated)
# vs SWE_RUN_NOACQ=1 (state read through L2 only; L1 keeps the geometry)
out=gpurun_out/r02_ab_noacq.txt
: > $out
one() {  # label cfg steps env...
  local lab=$1 cfg=$2 k=$3; shift 3
  env "$@" python bench.py --config $cfg --steps $k --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', '$lab', round(d['ms_per_step']*1e3,3), 'us/step', d['clocks']['sm_mhz'])" >> $out
}
for rep in 1 2; do
  one acq circular_dam_break 3000 SWE_RUN_NOACQ=0
  one noacq circular_dam_break 3000 SWE_RUN_NOACQ=1
  one acq three_mounds_friction 300 SWE_PERSISTENT=1 SWE_RUN_NOACQ=0
  one noacq three_mounds_friction 300 SWE_PERSISTENT=1 SWE_RUN_NOACQ=1
done
for p in 8 32; do
  for lab in "acq SWE_PERSISTENT=1 SWE_RUN_NOACQ=0" "noacq SWE_PERSISTENT=1 SWE_RUN_NOACQ=1"; do
    set -- $lab
    l=$1; shift
    echo "parts$p $l $(env "$@" timeout 300 python tools/run_timing.py --config channel --parts $p 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["us_per_step"],2), "us/step")')" >> $out
  done
done
