#!/bin/bash
# rotated tile schedule (SWE_TILE_ROT) vs plain round robin vs the previous build (exp/base_now)
out=gpurun_out/r02_ab_rot.txt
: > $out
one() {  # label cfg env...
  local lab=$1 cfg=$2; shift 2
  env "$@" python bench.py --config $cfg --steps 200 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', '$lab', round(d['ms_per_step']*1e3,2), 'us/step', 'tile', round(d['roofline']['kernel_ms']['tile']*1e3,2))" >> $out
}
for rep in 1 2; do
  for cfg in three_mounds_friction channel sloping_wet_dry; do
    one rot $cfg SWE_TILE_ROT=1
    one norot $cfg SWE_TILE_ROT=0
    one head $cfg SWE_B200_LIB=exp/base_now/libswe_b200.so
  done
done
for k in 0 3 1; do
  for lab in "rot SWE_TILE_ROT=1" "norot SWE_TILE_ROT=0"; do
    set -- $lab; l=$1; shift
    echo "part$k $l $(env "$@" timeout 300 python tools/_part_steps.py $k plain 2>&1 | tail -1)" >> $out
  done
done
