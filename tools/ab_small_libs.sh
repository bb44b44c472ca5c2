#!/bin/bash
# config [0] / [1] step times of experiment builds exp/<name>/ against the in-tree library
out=gpurun_out/r02_ab_small_libs.txt
: > $out
for rep in 1 2; do
  for lib in base "$@"; do
    e=""; [ $lib != base ] && e="SWE_B200_LIB=exp/$lib/libswe_b200.so"
    for cfg in circular_dam_break three_mounds_friction; do
      k=3000; [ $cfg = three_mounds_friction ] && k=300
      env $e SWE_PERSISTENT=1 python bench.py --config $cfg --steps $k --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null \
        | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', '$lib', round(d['ms_per_step']*1e3,3), 'us/step')" >> $out
    done
  done
done
