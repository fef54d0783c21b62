#!/bin/bash
# Per-layer MMA-thread wait breakdown for the 7 bench layers (round 2 diagnosis):
# full and MMA-only (CGB_DEBUG_SW=13: producers skip loads, filter TMA skipped, stores off),
# each with the per-CTA stats (bit 64).
for L in r50_3x3_56_64 r50_3x3_28_128 r50_3x3_14_256 r50_3x3_7_512 r50_3x3_s2_56_128 r50_3x3_s2_28_256 r50_3x3_s2_14_512; do
  R="timeout 60 python tools/run_layer.py --layer $L --reps 10"
  echo "=== $L"
  CGB_SW_VERBOSE=1 $R 2>&1 | grep -v "^\[cgb\] launch" | tail -2
  echo "-- full + stats"; CGB_DEBUG_SW=64 $R 2>&1 | tail -9
  echo "-- mma-only + stats"; CGB_DEBUG_SW=77 $R 2>&1 | tail -9
  echo "-- mma+tma (no loads, no stores) + stats"; CGB_DEBUG_SW=69 $R 2>&1 | tail -9
done
