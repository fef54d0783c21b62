#!/bin/bash
# Round-2 quick check on a GPU box: GPU parity suites, the bench step, per-layer diag.
# usage: tools/r02_check.sh [tests|bench|diag]...
for what in "$@"; do
  case $what in
    tests) timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/tests.log ;;
    bench) timeout 600 python bench.py --steps 20 --warmup 5 --quick --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?";
           python -c "import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print('step ms', round(d['ms_per_step'],4), 'TFLOPS', round(d['roofline']['achieved'],1), [ (l['layer'][8:], l['ms']) for l in d['roofline']['per_layer']], d['clocks'])" ;;
    diag) bash tools/diag_all.sh > gpurun_out/diag.log 2>&1; echo "diag rc=$?" ;;
  esac
done
