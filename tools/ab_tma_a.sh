# 1x1 layers (C3 geometries): TMA-fed A (default) vs producer staging (CGB_SW_TMA_A=0)
for rep in 1 2; do for e in 1 0; do
  for g in "256 1 64 56 1 0 256" "256 1 1024 14 1 0 256" "512 1 2048 7 1 0 256" "2048 1 512 7 1 0 256"; do
    echo "tma_a=$e $(CGB_SW_TMA_A=$e timeout 60 python tools/time_geom.py $g | tail -1)"
  done
done; done
