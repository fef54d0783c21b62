#!/bin/bash
# Filter-ring depth: default config vs deeper B-stage variants of the same tile shape.
run() { CGB_SW_VERBOSE=1 timeout 60 python tools/run_layer.py --layer $1 --reps 20 2>&1 | grep -E "launch|TFLOPS" | tail -2 | tr '\n' ' '; echo; }
for x in "r50_3x3_56_64:36" "r50_3x3_28_128:37" "r50_3x3_14_256:38" "r50_3x3_7_512:40" "r50_3x3_s2_56_128:41" "r50_3x3_s2_28_256:39" "r50_3x3_s2_14_512:39"; do
  l=${x%%:*}; c=${x##*:}
  echo -n "default "; run $l
  echo -n "cfg $c  "; CGB_SW_CFG=$c run $l
done
