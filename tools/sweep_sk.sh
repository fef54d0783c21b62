#!/bin/bash
# Time each BASELINE layer at every M tile with stream-K auto (SK=1) and forced (SK=2).
for l in ${LAYERS:-r50_3x3_56_64 r50_3x3_28_128 r50_3x3_14_256 r50_3x3_7_512 r50_3x3_s2_56_128 r50_3x3_s2_28_256 r50_3x3_s2_14_512}; do
  for mt in ${MTS:-1 2 4}; do
    for sk in 1 2; do
      echo -n "$l mt=$mt sk=$sk pair=${CGB_SW_PAIR:-1} "; CGB_SW_SK=$sk CGB_SW_MT=$mt CGB_SW_VERBOSE=1 timeout 60 python tools/run_layer.py --layer $l --reps 20 2>&1 | grep -E "launch|TFLOPS" | tail -2 | sed 's/\[cgb\] //' | tr '\n' ' '; echo
    done
  done
done
