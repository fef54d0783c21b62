for l in r50_3x3_14_256 r50_3x3_7_512 r50_3x3_s2_28_256 r50_3x3_s2_14_512; do
  echo "== $l default: $(CGB_SW_VERBOSE=1 timeout 60 python tools/run_layer.py --layer $l --reps 20 2>&1 | grep -E 'cand|TFLOPS' | tail -2 | tr '\n' ' ')"
  for c in 10 11 12 35 36 37 25 27 28; do
    echo "   cfg $c: $(CGB_SW_CFG=$c CGB_SW_VERBOSE=1 timeout 60 python tools/run_layer.py --layer $l --reps 20 2>&1 | grep -E 'launch|TFLOPS' | tail -2 | sed 's/\[cgb\] launch //' | tr '\n' ' ')"
  done
done
