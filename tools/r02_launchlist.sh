#!/bin/bash
# ncu launch list of the bench command. The graph-replayed step (programmatic dependent
# launch edges between kernel nodes) makes ncu report LaunchFailed on its third node; the
# same command with pdl=0 checks that hypothesis.
mkdir -p gpurun_out/r02
CMD="python bench.py --steps 2 --warmup 3 --quick --no-cpu-baseline --no-parity"
K='regex:sw_conv|splitk|tc_gather|tc_conv|im2col|ffma|filter_prep|k2_'
$CMD --tune '{"pdl":0}' > gpurun_out/r02/plain_nopdl.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 80 --csv --log-file gpurun_out/r02/launches_nopdl.csv \
    $CMD --tune '{"pdl":0}' > gpurun_out/r02/ncu_launch_nopdl.log 2>&1
echo "launch list (pdl=0) rc=$?"
ncu --graph-profiling node --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 80 --csv --log-file gpurun_out/r02/launches_graphnode.csv \
    $CMD > gpurun_out/r02/ncu_launch_graphnode.log 2>&1
echo "launch list (graph-profiling node) rc=$?"
tail -3 gpurun_out/r02/launches_nopdl.csv | cut -c1-200
