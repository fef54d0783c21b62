#!/bin/bash
# Stream-K (CGB_SW_SK=1 auto) against whole tiles only (0), per BASELINE layer.
for l in r50_3x3_56_64 r50_3x3_28_128 r50_3x3_14_256 r50_3x3_7_512 r50_3x3_s2_56_128 r50_3x3_s2_28_256 r50_3x3_s2_14_512; do
  for sk in 1 0; do
    echo -n "sk=$sk "; CGB_SW_SK=$sk CGB_SW_VERBOSE=1 timeout 60 python tools/run_layer.py --layer $l --reps 20 2>&1 | tail -2 | tr '\n' ' '; echo
  done
  for mt in ${MTS:-}; do echo -n "sk=1 mt=$mt "; CGB_SW_MT=$mt CGB_SW_VERBOSE=1 timeout 60 python tools/run_layer.py --layer $l --reps 20 2>&1 | tail -2 | tr '\n' ' '; echo; done
done
