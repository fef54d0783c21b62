# FFMA kernel (K4): current build vs a reference build (CGB_LIB_OVERRIDE=$1), fused and explicit
for rep in 1 2; do for lib in "" $1; do
  for g in "64 3 64 56 1 1 8" "64 7 3 224 2 3 8" "256 1 64 56 1 0 16"; do
    echo "${lib:-current} $(CGB_LIB_OVERRIDE=$lib timeout 60 python tools/time_geom.py $g ffma 2>&1 | tail -1)"
  done
done; done
