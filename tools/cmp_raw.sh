#!/bin/bash
# TMA-fed producers (CGB_SW_RAW=1) against register-staged LDG producers, per layer and config.
run() { timeout 60 python tools/run_layer.py --layer $1 --reps 20 2>&1 | grep -E "launch|TFLOPS" | tail -2 | tr '\n' ' '; echo; }
for l in ${LAYERS:-r50_3x3_56_64 r50_3x3_28_128 r50_3x3_14_256 r50_3x3_s2_56_128 r50_3x3_s2_28_256 r50_3x3_s2_14_512}; do
  echo "### $l"
  echo -n "ldg     "; CGB_SW_VERBOSE=1 run $l
  echo -n "raw     "; CGB_SW_RAW=1 CGB_SW_VERBOSE=1 run $l
  for c in ${CFGS:-31 32 33 34 35}; do echo -n "raw c$c "; CGB_SW_CFG=$c CGB_SW_RAW=1 CGB_SW_VERBOSE=1 run $l; done
  echo -n "raw prod-only "; CGB_DEBUG_SW=14 CGB_SW_RAW=1 run $l
done
