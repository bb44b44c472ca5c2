#!/bin/bash
# A/B of library variants built under exp/<name>/ (one line per run):
# tools/ab.sh "v1 v2" "channel sloping_wet_dry three_mounds_friction" [reps] [steps]
libs="$1"; cfgs="${2:-channel}"; reps=${3:-2}; steps=${4:-200}
for r in $(seq $reps); do
  for c in $cfgs; do
    for v in $libs; do
      SWE_B200_LIB=exp/$v/libswe_b200.so timeout 300 python tools/exp_step.py --config $c --steps $steps > gpurun_out/ab.json 2>&1
      echo "$v $c $(python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(round(d['graph_ms_per_step_1'],4), {k:round(v,4) for k,v in d['kernel_ms'].items()})" 2>&1 | tail -1)"
    done
  done
done
