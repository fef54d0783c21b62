#!/bin/bash
# Evidence for profiles/: plain bench run, then the ncu launch list of the same command
# (our kernels only), then one --set full capture per hot kernel. Run under gpurun.
set -x
CMD="python bench.py --steps 3 --warmup 3 --quick --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"sw_conv|tc_gather|tc_conv|im2col|ffma|filter_prep" -c 70 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
for L in "$@"; do
  python tools/run_layer.py --layer $L --reps 3 > gpurun_out/plain_$L.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"sw_conv|tc_gather" -s 2 -c 1 \
      -o gpurun_out/prof_$L python tools/run_layer.py --layer $L --reps 3 > gpurun_out/ncu_$L.log 2>&1
done
