#!/bin/bash
# Round-2 evidence (product build unless noted): all-config timings, simulator CSVs,
# workspace demo, cold-cache ncu of the explicit path and fc6 with the final kernels.
export CGB_LIB_OVERRIDE=$PWD/paper_2005_06410_b200/libconvgemm_b200.so
mkdir -p gpurun_out/ev
python tools/bench_configs.py --out gpurun_out/ev/r02_configs.json > gpurun_out/ev/configs.log 2>&1; echo "configs rc=$?"; tail -8 gpurun_out/ev/configs.log
for P in tf32 auto; do
  python tools/simulate.py --batch 64 --algo convgemm --precision $P --check --out gpurun_out/ev > gpurun_out/ev/sim_$P.log 2>&1; echo "sim $P rc=$?"; cat gpurun_out/ev/sim_$P.log | tail -2
done
python tools/simulate.py --batch 64 --algo im2col --precision tf32 --models vgg16 --out gpurun_out/ev > gpurun_out/ev/sim_im2col.log 2>&1; echo "sim im2col rc=$?"; tail -1 gpurun_out/ev/sim_im2col.log
python tools/workspace_demo.py --out gpurun_out/ev/r02_workspace.json > gpurun_out/ev/workspace.log 2>&1; echo "workspace rc=$?"; tail -5 gpurun_out/ev/workspace.log
bash tools/r02_explicit_ncu.sh
