#!/bin/bash
# Same-box A/B of the bench step: alternate bench.py runs with different --tune JSON.
# usage: tools/ab_bench.sh ROUNDS '{}' '{"tps":1}' ...
R=$1; shift
for r in $(seq 1 $R); do
  for v in "$@"; do
    python bench.py --steps 20 --warmup 5 --quick --no-cpu-baseline --tune "$v" 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step']*1e3,1), d['clocks']['sm_mhz'], ' '.join(str(round(l['ms']*1e3,1)) for l in d['roofline']['per_layer']))"
  done
done
