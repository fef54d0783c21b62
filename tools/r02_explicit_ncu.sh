#!/bin/bash
# ncu --set full of the explicit path's kernels (cold caches): K1 + K2 (TF32), K2 (3xTF32), fc6
mkdir -p gpurun_out/r02x
for CS in explicit:2 explicit3x:3 fc6:2; do
  C=${CS%%:*}; S=${CS##*:}
  python tools/ncu_cases.py $C > gpurun_out/r02x/plain_$C.log 2>&1 && \
  ncu --set full --cache-control all --clock-control none --import-source on \
      -k regex:"k2_|im2col|filter_prep" -s $S -c $S \
      -o gpurun_out/r02x/case_$C python tools/ncu_cases.py $C > gpurun_out/r02x/ncu_$C.log 2>&1
  echo "$C rc=$?"
done
for f in gpurun_out/r02x/*.ncu-rep; do
  python tools/ncu_summary.py $f > ${f%.ncu-rep}_raw.txt 2>&1
  python tools/ncu_stalls.py $f 30 > ${f%.ncu-rep}_hot.txt 2>&1
done
rm -f gpurun_out/r02x/case_fc6.ncu-rep
du -sh gpurun_out/r02x
