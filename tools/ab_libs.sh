#!/bin/bash
# A/B of library variants (exp/<name>/libswe_b200.so) x env settings on bench.py
# usage: tools/ab_libs.sh out.txt "name[:ENV=V,...]" ... ; configs in $CFGS (default channel)
out=$1; shift
CFGS=${CFGS:-channel}
: > $out
for rep in 1 2; do
for cfg in $CFGS; do
  for v in "$@"; do
    name=${v%%:*}; envs=""; [[ "$v" == *:* ]] && envs=${v#*:}
    env SWE_B200_LIB=exp/$name/libswe_b200.so ${envs//,/ } timeout 600 python bench.py --config $cfg --steps 200 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); L=d['roofline']['layout']; print('$cfg', '$v', 'rep$rep', round(d['ms_per_step']*1e3,2), 'us/step tile', round(d['roofline']['kernel_ms']['tile']*1e3,2), 'T', L['tile_cells'], 'grid', L['grid_tile'], 'smem', L['tile_smem_bytes'])" >> $out
  done
done
done
