#!/bin/bash
# A/B an environment switch per BASELINE layer: tools/ab_env.sh "A_ENV" "B_ENV" (e.g. "" "CGB_DEBUG_SW=128").
# Alternates A and B twice per layer (same box) to expose run-to-run noise.
A="$1"; B="$2"
for l in ${LAYERS:-r50_3x3_56_64 r50_3x3_28_128 r50_3x3_14_256 r50_3x3_7_512 r50_3x3_s2_56_128 r50_3x3_s2_28_256 r50_3x3_s2_14_512}; do
  for rep in 1 2; do
    for v in A B; do
      if [ $v = A ]; then E="$A"; else E="$B"; fi
      echo -n "$l $v "; env $E timeout 60 python tools/run_layer.py --layer $l --reps 20 --batch ${BATCH:-128} 2>&1 | grep TFLOPS
    done
  done
done
