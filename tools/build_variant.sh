#!/bin/bash
# Build a profiling variant of the library: tools/build_variant.sh NAME -DFLAG=... ...
name=$1; shift
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  "$@" paper_2005_06410_b200/csrc/*.cu -o tools/libcgb_$name.so 2>&1 | grep -E "error|spill" | sort | uniq -c | sort -rn | head -3
