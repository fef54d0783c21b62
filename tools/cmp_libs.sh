#!/bin/bash
for lib in "" tools/libcgb_ldg1.so tools/libcgb_ldg2.so; do
  echo "== lib=${lib:-default}"
  for l in r50_3x3_56_64 r50_3x3_28_128 r50_3x3_s2_56_128 r50_3x3_s2_28_256 r50_3x3_s2_14_512; do
    CGB_LIB_OVERRIDE=$lib timeout 60 python tools/run_layer.py --layer $l --reps 10 2>&1 | tail -1
    CGB_DEBUG_SW=14 CGB_LIB_OVERRIDE=$lib timeout 60 python tools/run_layer.py --layer $l --reps 10 2>&1 | tail -1 | sed 's/^/   producer-only: /'
  done
done
