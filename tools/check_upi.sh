for c in "" 0 38; do echo "vgg2 cfg=$c $(CGB_SW_CFG=$c timeout 60 python tools/time_geom.py 64 3 64 224 1 1 64 | tail -1)"; done
for c in "" 0 38; do echo "c1 cfg=$c $(CGB_SW_CFG=$c timeout 60 python tools/time_geom.py 64 3 64 56 1 1 8 | tail -1)"; done
for i in 1 2 3; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --quick 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'], [l['ms'] for l in d['roofline']['per_layer']])"; done
