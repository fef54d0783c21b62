#!/bin/bash
# Cold-cache ncu --set full of the 7 bench layers on the final build (product library), then
# the raw / hot summaries; the .ncu-rep of the two weakest layers are kept.
export CGB_LIB_OVERRIDE=$PWD/paper_2005_06410_b200/libconvgemm_b200.so
mkdir -p gpurun_out/r02
for L in r50_3x3_56_64 r50_3x3_28_128 r50_3x3_14_256 r50_3x3_7_512 r50_3x3_s2_56_128 r50_3x3_s2_28_256 r50_3x3_s2_14_512; do
  python tools/run_layer.py --layer $L --reps 1 --warm 1 > gpurun_out/r02/plain_$L.log 2>&1 && \
  ncu --set full --cache-control all --clock-control none --import-source on -k regex:"sw_conv" -s 1 -c 1 \
      -o gpurun_out/r02/prof_$L -f python tools/run_layer.py --layer $L --reps 1 --warm 1 > gpurun_out/r02/ncu_$L.log 2>&1
  echo "$L rc=$?"
  python tools/ncu_summary.py gpurun_out/r02/prof_$L.ncu-rep > gpurun_out/r02/prof_${L}_raw.txt 2>&1
  python tools/ncu_stalls.py gpurun_out/r02/prof_$L.ncu-rep 30 > gpurun_out/r02/prof_${L}_hot.txt 2>&1
  grep -E "gpu__time_duration|dram__bytes|tensor_cycles" gpurun_out/r02/prof_${L}_raw.txt
done
for f in gpurun_out/r02/*.ncu-rep; do
  case "$f" in *s2_56_128*|*56_64*) ;; *) rm -f "$f" ;; esac
done
