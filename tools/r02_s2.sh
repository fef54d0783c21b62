#!/bin/bash
# s2 56->28 c128: filter-stage group sizes and ring depths (profiling build)
L=${L:-r50_3x3_s2_56_128}
for c in 40 50 6 41; do for t in 0 1 2 3; do
  echo -n "cand $c tps $t: "; CGB_SW_CFG=$c CGB_SW_TPS=$t CGB_DEBUG_SW=64 timeout 60 python tools/run_layer.py --layer $L --reps 10 2>&1 | grep -E "MMA thread|TFLOPS" | sed -e 's/epilogue.*//' | tr '\n' ' '; echo
done; done
