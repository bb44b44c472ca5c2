#!/bin/bash
# config [0] tile-size sweep of the persistent kernel (long windows)
out=gpurun_out/r02_sweep_small2.txt
: > $out
for rep in 1 2; do
for T in default 32 48 64 80; do
  if [ $T = default ]; then e=""; else e="SWE_TILE_CELLS=$T"; fi
  env $e python bench.py --config circular_dam_break --steps 3000 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); l=d['roofline']['layout']; print('$T', round(d['ms_per_step']*1e3,3), 'us/step', 'T', l.get('tile_cells'), 'tiles', l.get('tiles'))" >> $out
done
done
