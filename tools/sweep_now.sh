# candidate sweep on the current build: VGG conv1 / stem (time_geom) and the two staging-bound layers
for c in "" 0 1 2 38 39; do echo "vgg1 cfg=$c $(CGB_SW_CFG=$c timeout 60 python tools/time_geom.py 64 3 3 224 1 1 64 | tail -1)"; done
for c in "" 0 1 2 38 39; do echo "stem cfg=$c $(CGB_SW_CFG=$c timeout 60 python tools/time_geom.py 64 7 3 224 2 3 256 | tail -1)"; done
LC="r50_3x3_56_64:0,1,31,38,39,14 r50_3x3_s2_56_128:5,6,7,33,34,40,41" bash tools/sweep_probe.sh
