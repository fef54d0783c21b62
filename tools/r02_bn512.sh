timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "bn512" 2>&1 | tail -5
for g in "512 1 2048 7 1 0 256" "2048 1 512 7 1 0 256"; do
  for rep in 1 2; do
  echo -n "default "; timeout 60 python tools/time_geom.py $g 2>&1 | tail -1
  for c in 54 55; do echo -n "bn512 cfg=$c "; CGB_SW_BN=512 CGB_SW_CFG=$c timeout 60 python tools/time_geom.py $g 2>&1 | tail -1; done
  done
  CGB_SW_BN=512 CGB_SW_CFG=54 CGB_SW_VERBOSE=1 timeout 60 python tools/time_geom.py $g 2>&1 | grep "\[cgb\] launch" | tail -1 | cut -c1-140
done
