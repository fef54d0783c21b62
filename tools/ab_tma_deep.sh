# 1x1 TMA-fed A: deep A rings (default) vs the regular table (CGB_SW_TMA_DEEP=0)
for rep in 1 2; do for e in 1 0; do
  for g in "256 1 64 56 1 0 256" "256 1 1024 14 1 0 256"; do
    echo "deep=$e $(CGB_SW_TMA_DEEP=$e CGB_SW_VERBOSE=1 timeout 60 python tools/time_geom.py $g 2>&1 | grep -E 'cand|TFLOPS' | tail -2 | tr '\n' ' ')"
  done
done; done
