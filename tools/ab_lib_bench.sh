# same-box A/B of a library variant on the bench step: tools/ab_lib_bench.sh tools/libcgb_X.so [steps]
V=$1; S=${2:-200}
for rep in 1 2; do for lib in "" $V; do
  echo -n "${lib:-default} "; CGB_LIB_OVERRIDE=$lib python bench.py --quick --no-cpu-baseline --steps $S 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'], [l['ms'] for l in d['roofline']['per_layer']])"
done; done
