#!/bin/bash
# A/B of one environment switch of the in-tree library: tools/ab_env.sh <name> "<ENV=..>" [configs...]
name=$1; envs=$2; shift 2
cfgs=${@:-channel sloping_wet_dry three_mounds_friction}
out=gpurun_out/r02_ab_$name.txt
: > $out
one() {  # label cfg env...
  local lab=$1 cfg=$2; shift 2
  env "$@" python bench.py --config $cfg --steps 200 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', '$lab', round(d['ms_per_step']*1e3,2), 'us/step', 'tile', round(d['roofline']['kernel_ms']['tile']*1e3,2), d['clocks']['sm_mhz'])" >> $out
}
for rep in 1 2; do
  for cfg in $cfgs; do
    one base $cfg $envs
    one $name $cfg
  done
done
