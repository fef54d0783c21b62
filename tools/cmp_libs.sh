#!/bin/bash
for lib in "" tools/libcgb_pw12.so tools/libcgb_pw16.so; do
  echo "== lib=${lib:-default}"
  for l in r50_3x3_56_64 r50_3x3_28_128 r50_3x3_14_256 r50_3x3_7_512 r50_3x3_s2_56_128 r50_3x3_s2_28_256 r50_3x3_s2_14_512; do
    CGB_LIB_OVERRIDE=$lib timeout 60 python tools/run_layer.py --layer $l --reps 10 2>&1 | tail -1
  done
done
