# 7x7 1x1 layers (staged, not TMA-eligible): default vs the deep-A-ring candidate 48
for rep in 1 2; do for c in "" 48; do
  for g in "512 1 2048 7 1 0 256" "2048 1 512 7 1 0 256"; do
    echo "cfg=$c $(CGB_SW_CFG=$c CGB_SW_VERBOSE=1 timeout 60 python tools/time_geom.py $g 2>&1 | grep -E 'launch|TFLOPS' | tail -2 | sed 's/\[cgb\] launch //' | tr '\n' ' ')"
  done
done; done
