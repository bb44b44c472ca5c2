for c in "channel --parts 8" "channel --parts 4" "three_mounds_friction"; do
  echo "tim $(SWE_PERSISTENT=1 SWE_B200_LIB=exp/tim/libswe_b200.so timeout 300 python tools/run_timing.py --config $c 2>&1 | tail -1)"
  echo "graph $(SWE_PERSISTENT=0 timeout 300 python tools/run_timing.py --config $c 2>&1 | tail -1)"
done > gpurun_out/r02_run_timing.txt
