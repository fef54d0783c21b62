#!/bin/bash
# MMA-only (CGB_DEBUG_SW=77) and full cycle counts per candidate configuration.
run() { L=$1; shift; for c in "$@"; do
  for m in 64 77; do
    echo -n "$L cand $c dbg $m: "; CGB_SW_CFG=$c CGB_DEBUG_SW=$m timeout 60 python tools/run_layer.py --layer $L --reps 10 2>&1 | grep -E "MMA thread|TFLOPS" | tr '\n' ' ' ; echo
  done; done; }
run r50_3x3_s2_56_128 40 6 7 5 41 33 34 21 19
run r50_3x3_28_128 5 6 7 41 40 19 21
run r50_3x3_56_64 0 1 2 38 39 14 15 16
