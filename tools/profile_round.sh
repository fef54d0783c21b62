#!/bin/bash
# Evidence for profiles/: plain bench run, then the ncu launch list of the same command
# (our kernels only), then one --set full capture per BASELINE layer (TF32). Run under
# gpurun on one GPU; each ncu command runs only after the same command exited 0 without ncu.
set -x
CMD="python bench.py --steps 3 --warmup 3 --quick --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"sw_conv|tc_gather|tc_conv|im2col|ffma|filter_prep" -c 80 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
LAYERS=${LAYERS:-"r50_3x3_56_64 r50_3x3_28_128 r50_3x3_14_256 r50_3x3_7_512 r50_3x3_s2_56_128 r50_3x3_s2_28_256 r50_3x3_s2_14_512"}
for L in $LAYERS; do
  python tools/run_layer.py --layer $L --reps 3 > gpurun_out/plain_$L.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"sw_conv|tc_gather" -s 2 -c 1 \
      -o gpurun_out/prof_$L python tools/run_layer.py --layer $L --reps 3 > gpurun_out/ncu_$L.log 2>&1
done
ls -la gpurun_out/
# summarise on the box (gpurun copies back at most 64 MiB): text evidence into
# gpurun_out/prof_txt/, keep one full report, drop the rest
python tools/make_profiles.py r01 gpurun_out/prof_txt > gpurun_out/prof_txt.log 2>&1
for f in gpurun_out/prof_*.ncu-rep; do
  case "$f" in *s2_56_128*) ;; *) rm -f "$f" ;; esac
done
du -sh gpurun_out
