#!/bin/bash
# Bounds-checked build of the library (device-side SWE_CHECK traps on any
# out-of-range tile / cell / edge / shared-memory slot / halo index), the
# stand-in for compute-sanitizer, which is closed on this GPU pool.
#   tools/checked_build.sh && SWE_B200_LIB=exp/checked/libswe_b200.so python -m pytest tests -m gpu
set -e
cd "$(dirname "$0")/.."
mkdir -p exp/checked
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude -Ipaper_1807_00672_b200/csrc \
  -DSWE_CHECKED=1 -c paper_1807_00672_b200/csrc/swe_dev.cu -o exp/checked/swe_dev.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o exp/checked/libswe_b200.so \
  exp/checked/swe_dev.o paper_1807_00672_b200/_build/host_abi.o
