#!/bin/bash
# persistent-kernel experiments on the 10M channel (SWE_* env / build variants)
out=gpurun_out/r02_exp_persist.txt
: > $out
run() {  # label, env...
  local lab=$1; shift
  env "$@" python bench.py --config channel --steps 200 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lab', round(d['ms_per_step']*1e3,2), 'us/step', d['roofline']['layout']['grid_run'])" >> $out
}
run base_persist SWE_PERSISTENT=1
run base_graph SWE_PERSISTENT=0
run noskip_persist SWE_PERSISTENT=1 SWE_NO_DRY_SKIP=1
run noskip_graph SWE_PERSISTENT=0 SWE_NO_DRY_SKIP=1
if [ -f exp/nc/libswe_b200.so ]; then
  run nc_persist SWE_PERSISTENT=1 SWE_B200_LIB=exp/nc/libswe_b200.so
  run nc_noskip_persist SWE_PERSISTENT=1 SWE_NO_DRY_SKIP=1 SWE_B200_LIB=exp/nc/libswe_b200.so
fi
