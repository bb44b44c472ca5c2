timeout 300 python -m pytest tests/test_gpu_persistent.py -q -x --timeout 120 > gpurun_out/r02_persist_a.log 2>&1; echo rc=$? >> gpurun_out/r02_persist_a.log
timeout 1500 tools/ab_persist.sh
