#!/bin/bash
# Per-layer breakdown: full, MMA-only (skip loads/stores/TMA), MMA+TMA, producer-only, stats.
L=${1:-r50_3x3_7_512}
R="timeout 60 python tools/run_layer.py --layer $L --reps 10"
CGB_SW_VERBOSE=1 $R 2>&1 | tail -2
echo -n "mma-only      "; CGB_DEBUG_SW=13 $R 2>&1 | tail -1
echo -n "mma+tma       "; CGB_DEBUG_SW=5 $R 2>&1 | tail -1
echo -n "no-stores     "; CGB_DEBUG_SW=4 $R 2>&1 | tail -1
echo -n "producer-only "; CGB_DEBUG_SW=14 $R 2>&1 | tail -1
CGB_DEBUG_SW=64 $R 2>&1 | tail -2
for c in ${CFGS:-}; do echo -n "cfg $c "; CGB_SW_CFG=$c $R 2>&1 | tail -1; done
