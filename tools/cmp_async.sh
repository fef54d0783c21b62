#!/bin/bash
# Compare cp.async window fill (CGB_SW_ASYNC=1) against register-staged fill (=0).
for as in 1 0; do
  echo "== CGB_SW_ASYNC=$as"
  for l in r50_3x3_56_64 r50_3x3_28_128 r50_3x3_14_256 r50_3x3_7_512 r50_3x3_s2_56_128 r50_3x3_s2_28_256 r50_3x3_s2_14_512; do
    CGB_SW_ASYNC=$as timeout 60 python tools/run_layer.py --layer $l --reps 10 2>&1 | tail -1
    CGB_SW_ASYNC=$as CGB_DEBUG_SW=14 timeout 60 python tools/run_layer.py --layer $l --reps 10 2>&1 | tail -1 | sed 's/^/   producer-only: /'
  done
done
