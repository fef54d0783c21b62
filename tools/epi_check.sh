# quick A/B helper: stem, VGG conv1 and the bench step (3 runs)
for g in "64 7 3 224 2 3 256" "64 3 3 224 1 1 64" "64 3 64 56 1 1 128" "128 3 128 56 2 1 128"; do
  timeout 60 python tools/time_geom.py $g 2>&1 | tail -1
done
for i in 1 2 3; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --quick 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'], [l['ms'] for l in d['roofline']['per_layer']])"; done
