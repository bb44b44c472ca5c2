#!/bin/bash
# run tools/exp_step.py over library variants x modes; one line per run
# usage: tools/exp_matrix.sh "lib1 lib2 ..." "mode args ..." [presteps]
libs="$1"; shift
modes="$1"; shift
pre=${1:-0}
for lib in $libs; do
  IFS=';' read -ra MS <<< "$modes"
  for m in "${MS[@]}"; do
    env $m timeout 300 python tools/exp_step.py --steps 100 --presteps $pre $( [[ "$m" == *TWO* ]] && echo --two-phase ) > gpurun_out/e.json 2>&1
    echo "$lib [$m] $(python -c "import json;d=json.load(open('gpurun_out/e.json'));print(round(d['graph_ms_per_step_1'],4), {k:round(v,4) for k,v in d['kernel_ms'].items()})" 2>&1 | tail -1)"
  done
done
