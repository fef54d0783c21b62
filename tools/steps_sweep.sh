# bench step time vs --steps on one box (mean of the per-step CUDA-event times), plus the per-step spread
for S in 20 200 20 200; do
  python bench.py --quick --no-cpu-baseline --steps $S 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print($S, round(d['ms_per_step']*1e3,1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
