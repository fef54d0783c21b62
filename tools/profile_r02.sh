#!/bin/bash
# Round-2 evidence for profiles/ (run under gpurun on one GPU): each ncu command runs
# only after the same command exited 0 without ncu. Product library (not the profiling
# build). Per-layer captures with --cache-control all: every replay pass starts from
# flushed caches, so dram bytes are the cold-cache traffic.
export CGB_LIB_OVERRIDE=$PWD/paper_2005_06410_b200/libconvgemm_b200.so
mkdir -p gpurun_out/r02
CMD="python bench.py --steps 2 --warmup 3 --quick --no-cpu-baseline --no-parity"
$CMD > gpurun_out/r02/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sw_conv|splitk|tc_gather|tc_conv|im2col|ffma|filter_prep" \
    -c 70 --csv --log-file gpurun_out/r02/launches.csv $CMD > gpurun_out/r02/ncu_launch.log 2>&1
echo "launch list rc=$?"
for L in r50_3x3_56_64 r50_3x3_28_128 r50_3x3_14_256 r50_3x3_7_512 r50_3x3_s2_56_128 r50_3x3_s2_28_256 r50_3x3_s2_14_512; do
  python tools/run_layer.py --layer $L --reps 1 --warm 1 > gpurun_out/r02/plain_$L.log 2>&1 && \
  ncu --set full --cache-control all --clock-control none --import-source on -k regex:"sw_conv" -s 1 -c 1 \
      -o gpurun_out/r02/prof_$L python tools/run_layer.py --layer $L --reps 1 --warm 1 > gpurun_out/r02/ncu_$L.log 2>&1
  echo "$L rc=$?"
done
for CS in explicit:2 ffma:1 fc6:1 stem:2 pw56:1; do
  C=${CS%%:*}; S=${CS##*:}  # kernels per iteration: skip the first iteration's
  python tools/ncu_cases.py $C > gpurun_out/r02/plain_$C.log 2>&1 && \
  ncu --set full --cache-control all --clock-control none --import-source on \
      -k regex:"sw_conv|tc_conv|im2col|ffma|filter_prep" -s $S -c $S \
      -o gpurun_out/r02/case_$C python tools/ncu_cases.py $C > gpurun_out/r02/ncu_$C.log 2>&1
  echo "$C rc=$?"
done
for f in gpurun_out/r02/*.ncu-rep; do
  python tools/ncu_summary.py $f > ${f%.ncu-rep}_raw.txt 2>&1
  python tools/ncu_stalls.py $f 30 > ${f%.ncu-rep}_hot.txt 2>&1
done
# keep the reports of the two weakest layers, drop the rest (64 MiB pull limit)
for f in gpurun_out/r02/*.ncu-rep; do
  case "$f" in *s2_56_128*|*56_64*) ;; *) rm -f "$f" ;; esac
done
du -sh gpurun_out/r02
