#!/bin/bash
# Time every shifted-window candidate config on each BASELINE layer (TF32).
for l in r50_3x3_56_64 r50_3x3_28_128 r50_3x3_14_256 r50_3x3_7_512 r50_3x3_s2_56_128 r50_3x3_s2_28_256 r50_3x3_s2_14_512; do
  for c in 0 1 2 5 6 7 8 11 12 13 14 15; do
    out=$(CGB_SW_CFG=$c timeout 60 python tools/run_layer.py --layer $l --reps 10 2>&1 | tail -1)
    echo "cfg=$c $out"
  done
done
