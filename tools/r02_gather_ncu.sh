#!/bin/bash
# cold-cache ncu --set full of the kernels outside the BASELINE geometries (AlexNet conv1 on
# the gather / reference-order path, AlexNet conv2's 25-tap shifted window)
export CGB_LIB_OVERRIDE=$PWD/paper_2005_06410_b200/libconvgemm_b200.so
mkdir -p gpurun_out/r02g
for C in ${CASES:-gather alex5}; do
  python tools/ncu_cases.py $C > gpurun_out/r02g/plain_$C.log 2>&1; cat gpurun_out/r02g/plain_$C.log | tail -1
  ncu --set full --cache-control all --clock-control none --import-source on \
      -k regex:"sw_conv|tc_conv|tc_gather|gather|ffma|filter_prep" -s 1 -c 2 \
      -o gpurun_out/r02g/case_$C python tools/ncu_cases.py $C > gpurun_out/r02g/ncu_$C.log 2>&1
  echo "$C rc=$?"
done
for f in gpurun_out/r02g/*.ncu-rep; do
  python tools/ncu_summary.py $f > ${f%.ncu-rep}_raw.txt 2>&1
  python tools/ncu_stalls.py $f 30 > ${f%.ncu-rep}_hot.txt 2>&1
done
rm -f gpurun_out/r02g/*.ncu-rep
head -24 gpurun_out/r02g/case_*_raw.txt
