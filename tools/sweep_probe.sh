#!/bin/bash
# Time candidate configurations (CGB_SW_CFG) on chosen layers: LC="layer:c1,c2 layer:c3"
for spec in ${LC}; do
  l=${spec%%:*}; cs=${spec#*:}
  echo "== $l default: $(CGB_SW_VERBOSE=1 timeout 60 python tools/run_layer.py --layer $l --reps 20 2>&1 | grep -E 'cand|TFLOPS' | tail -2 | tr '\n' ' ')"
  for c in ${cs//,/ }; do
    echo "   cfg $c: $(CGB_SW_CFG=$c CGB_SW_VERBOSE=1 timeout 60 python tools/run_layer.py --layer $l --reps 20 2>&1 | grep -E 'launch|TFLOPS' | tail -2 | sed 's/\[cgb\] launch //' | tr '\n' ' ')"
  done
done
