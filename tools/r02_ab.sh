#!/bin/bash
# same-box A/B of one tuning key on the bench step: tools/r02_ab.sh KEY [reps]
K=$1; N=${2:-3}
for rep in $(seq $N); do for v in 0 1; do
  python bench.py --steps 20 --warmup 5 --quick --no-cpu-baseline --no-parity --tune "{\"$K\":$v}" > gpurun_out/ab_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); print('$K=$v step us', round(d['ms_per_step']*1e3,1), [round(l['ms']*1e3,1) for l in d['roofline']['per_layer']], d['clocks']['sm_mhz'])"
done; done
