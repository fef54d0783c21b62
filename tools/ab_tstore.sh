# TMA-fed 1x1: TMA-store epilogue (default) vs register stores (CGB_SW_TSTORE=0)
for rep in 1 2; do for e in 1 0; do
  for g in "256 1 64 56 1 0 256" "256 1 1024 14 1 0 256" "128 1 256 28 1 0 128"; do
    echo "tstore=$e $(CGB_SW_TSTORE=$e timeout 60 python tools/time_geom.py $g 2>&1 | tail -1)"
  done
done; done
