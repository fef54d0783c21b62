# TMA-fed 1x1: 16 epilogue warps (default) vs 4 (CGB_DEBUG_SW=128)
for rep in 1 2; do for d in 0 128; do
  for g in "256 1 64 56 1 0 256" "256 1 64 56 1 0 64" "128 1 256 28 1 0 128"; do
    echo "dbg=$d $(CGB_DEBUG_SW=$d timeout 60 python tools/time_geom.py $g 2>&1 | tail -1)"
  done
done; done
