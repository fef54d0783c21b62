# same-box A/B of the bench's L2 policy at the default step count (clocks sampled in the timed region)
for rep in 1 2; do for m in flush cycle; do
  echo -n "$m "; python bench.py --quick --no-cpu-baseline --l2 $m 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'], [l['ms'] for l in d['roofline']['per_layer']])"
done; done
