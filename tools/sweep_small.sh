#!/bin/bash
# config [0] (10k cells): tile size / worker count / threads of the persistent kernel
out=gpurun_out/r02_sweep_small.txt
: > $out
one() {  # label env...
  local lab=$1; shift
  env "$@" python bench.py --config circular_dam_break --steps 3000 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); l=d['roofline']['layout']; print('$lab', round(d['ms_per_step']*1e3,3), 'us/step', 'T', l.get('tile_cells'), 'tiles', l.get('tiles'), 'grid_run', l['grid_run'])" >> $out
}
one default
for T in 32 48 64 96 128; do one T$T SWE_TILE_CELLS=$T; done
for G in 16 32 48 96; do one G$G SWE_RUN_GRID=$G; done
for G in 16 32 48; do one T64_G$G SWE_TILE_CELLS=64 SWE_RUN_GRID=$G; done
one thr256 SWE_TILE_THREADS=256
one thr256_T64 SWE_TILE_THREADS=256 SWE_TILE_CELLS=64
one default_again
