#!/bin/bash
# Stage breakdown of the low-channel layers (profiling build, CGB_DEBUG_SW bits:
# 1 no staging loads, 2 no MMAs, 4 no stores, 8 no filter TMA, 16 no epilogue loop)
for g in "64 7 3 224 2 3 256" "64 3 3 224 1 1 64"; do
  for d in 0 1 2 4 16 20 21 22 3 23 64; do echo -n "dbg=$d "; CGB_DEBUG_SW=$d timeout 60 python tools/time_geom.py $g 2>&1 | tail -${TAILN:-1}; done
done
