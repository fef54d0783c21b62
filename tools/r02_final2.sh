#!/bin/bash
# Final round-2 evidence after the last code change: the driver's sequence (r02_final.sh), the
# supplementary forked-stream steps, shard steps, per-CTA timelines at b=128 and b=16,
# the ncu launch list of the bench command and all-config / simulator numbers.
bash tools/r02_final.sh
bash tools/r02_conc.sh
bash tools/r02_shards.sh
mkdir -p gpurun_out/final
python tools/graph_timeline.py 2>&1 | grep -E "^entry|^ +mma end|^total" > gpurun_out/final/graph_timeline_b128.txt
TL_BATCH=16 python tools/graph_timeline.py 2>&1 | grep -E "^entry|^ +mma end|^total" > gpurun_out/final/graph_timeline_b16.txt
tail -1 gpurun_out/final/graph_timeline_b128.txt gpurun_out/final/graph_timeline_b16.txt
export CGB_LIB_OVERRIDE=$PWD/paper_2005_06410_b200/libconvgemm_b200.so
CMD="python bench.py --steps 2 --warmup 3 --quick --no-cpu-baseline --no-parity --concurrent="
$CMD > gpurun_out/final/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sw_conv|splitk|tc_gather|tc_conv|im2col|ffma|filter_prep" \
    -c 70 --csv --log-file gpurun_out/final/launches.csv $CMD > gpurun_out/final/ncu_launch.log 2>&1
echo "launch list rc=$? launches=$(grep -c sw_conv gpurun_out/final/launches.csv)"
python tools/bench_configs.py --out gpurun_out/final/r02_configs.json > gpurun_out/final/configs.log 2>&1; echo "configs rc=$?"; tail -7 gpurun_out/final/configs.log
for P in tf32 auto; do
  python tools/simulate.py --batch 64 --algo convgemm --precision $P --check --out gpurun_out/final 2>&1 | tail -3
done
