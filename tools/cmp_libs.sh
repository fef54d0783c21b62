#!/bin/bash
# Time each BASELINE layer under alternative library builds (CGB_LIB_OVERRIDE).
LIBS=${LIBS:-""}
LAYERS=${LAYERS:-"r50_3x3_56_64 r50_3x3_28_128 r50_3x3_14_256 r50_3x3_7_512 r50_3x3_s2_56_128 r50_3x3_s2_28_256 r50_3x3_s2_14_512"}
for lib in "" $LIBS; do
  echo "== lib=${lib:-default}"
  for l in $LAYERS; do
    CGB_LIB_OVERRIDE=$lib timeout 60 python tools/run_layer.py --layer $l --reps 20 2>&1 | tail -1
    if [ -n "$PROD" ]; then CGB_DEBUG_SW=14 CGB_LIB_OVERRIDE=$lib timeout 60 python tools/run_layer.py --layer $l --reps 10 2>&1 | tail -1 | sed 's/^/   producer-only: /'; fi
  done
done
