#!/bin/bash
# Time each BASELINE layer at every M tile (stream-K auto) to fit the dispatcher's cost model.
for l in ${LAYERS:-r50_3x3_56_64 r50_3x3_28_128 r50_3x3_14_256 r50_3x3_7_512 r50_3x3_s2_56_128 r50_3x3_s2_28_256 r50_3x3_s2_14_512}; do
  for mt in 1 2 4; do
    echo -n "mt=$mt "; CGB_SW_MT=$mt CGB_SW_VERBOSE=1 timeout 60 python tools/run_layer.py --layer $l --reps 20 2>&1 | grep -E "launch|TFLOPS" | tail -2 | tr '\n' ' '; echo
  done
done
