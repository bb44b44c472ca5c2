for lib in exp/tim; do for c in channel three_mounds_friction circular_dam_break; do
  echo "$lib $(SWE_B200_LIB=$lib/libswe_b200.so timeout 300 python tools/run_timing.py --config $c 2>&1 | tail -1)"; done; done > gpurun_out/r02_run_timing.txt
timeout 300 python -m pytest tests/test_gpu_persistent.py -q -x --timeout 120 > gpurun_out/r02_persist_a.log 2>&1; echo rc=$? >> gpurun_out/r02_persist_a.log
timeout 300 python -m pytest tests/test_gpu_persistent.py -q -x --timeout 120 > gpurun_out/r02_persist_a.log 2>&1; echo rc=$? >> gpurun_out/r02_persist_a.log
timeout 1500 tools/ab_persist.sh
