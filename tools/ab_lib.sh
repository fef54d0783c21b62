#!/bin/bash
# Same-box A/B of two library builds on the bench step: tools/ab_lib.sh ROUNDS libA.so libB.so
R=$1; A=$2; B=$3
for r in $(seq 1 $R); do
  for L in $A $B; do
    CGB_LIB_OVERRIDE=$L python bench.py --steps 20 --warmup 5 --quick --no-cpu-baseline --no-parity 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $L)', round(d['ms_per_step']*1e3,1), d['clocks']['sm_mhz'], ' '.join(str(round(l['ms']*1e3,1)) for l in d['roofline']['per_layer']))"
  done
done
