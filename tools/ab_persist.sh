#!/bin/bash
# A/B of the run loop: persistent kernel (default) vs the CUDA-graph loop, per BASELINE config
out=gpurun_out/r02_ab_persist.txt
: > $out
for cfg in channel sloping_wet_dry three_mounds_friction circular_dam_break; do
  for P in 1 0; do
    for rep in 1 2; do
      SWE_PERSISTENT=$P python bench.py --config $cfg --steps 200 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null \
        | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', 'persistent=$P', 'rep$rep', round(d['ms_per_step']*1e3,2), 'us/step', round(d['value']/1e9,3), 'G/s', 'tile_ms', round(d['roofline']['kernel_ms']['tile']*1e3,2), d['clocks']['sm_mhz'], 'grids', d['roofline']['layout']['grid_tile'], d['roofline']['layout']['grid_run'], 'skip', round(d['dry_tile_skip']['skipped_tile_fraction'],3))" >> $out
    done
  done
done
