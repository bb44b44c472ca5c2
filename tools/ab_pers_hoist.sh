#!/bin/bash
out=gpurun_out/r02_ab_pers_hoist.txt
: > $out
for rep in 1 2; do
  for lib in new base_now; do
    e=""; [ $lib != new ] && e="SWE_B200_LIB=exp/$lib/libswe_b200.so"
    for cs in "three_mounds_friction 1.0 300" "sloping_wet_dry 0.2 500" "circular_dam_break 1.0 3000"; do
      set -- $cs
      env $e SWE_PERSISTENT=1 python bench.py --config $1 --scale $2 --steps $3 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null \
        | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', '$2', '$lib', round(d['ms_per_step']*1e3,3), 'us/step')" >> $out
    done
  done
done
