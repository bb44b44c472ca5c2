#!/bin/bash
# An experiment build of the library with extra defines, into exp/<name>/:
#   tools/variant_build.sh tim -DSWE_RUN_TIMING=1
#   SWE_B200_LIB=exp/tim/libswe_b200.so python tools/run_timing.py --config circular_dam_break
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p exp/$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude -Ipaper_1807_00672_b200/csrc \
  "$@" -c paper_1807_00672_b200/csrc/swe_dev.cu -o exp/$name/swe_dev.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o exp/$name/libswe_b200.so \
  exp/$name/swe_dev.o paper_1807_00672_b200/_build/host_abi.o
