#!/bin/bash
# tile-size sweep of the graph loop at the current kernel (channel, dry bed)
out=gpurun_out/r02_sweep_T.txt
: > $out
for cfg in channel sloping_wet_dry; do
  for T in 224 192 208 216 232 240 256 224; do
    SWE_TILE_CELLS=$T python bench.py --config $cfg --steps 200 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', 'T=$T', round(d['ms_per_step']*1e3,2), 'us/step', 'tile', round(d['roofline']['kernel_ms']['tile']*1e3,2))" >> $out
  done
done
