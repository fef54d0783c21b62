# TMA-fed 1x1: A-ring depth probes (CGB_SW_CFG) on the two eligible C3 layers
for c in "" 48 50 51 52; do
  for g in "256 1 64 56 1 0 256" "256 1 1024 14 1 0 256"; do
    echo "cfg=$c $(CGB_SW_CFG=$c CGB_SW_VERBOSE=1 timeout 60 python tools/time_geom.py $g 2>&1 | grep -E 'launch|TFLOPS' | tail -2 | sed 's/\[cgb\] launch //' | tr '\n' ' ')"
  done
done
