#!/bin/bash
# AlexNet through the simulator (tests + b=64 sweeps with the conv_direct check on)
mkdir -p gpurun_out/alex
python -m pytest tests/test_simulator.py -q -m gpu -k "alexnet" 2>&1 | tail -5 > gpurun_out/alex/tests.txt
cat gpurun_out/alex/tests.txt
for p in tf32 auto; do
  python tools/simulate.py --models alexnet --batch 64 --precision $p --check --out gpurun_out/alex 2>&1 | tail -3
done
python tools/simulate.py --models alexnet --batch 64 --algo im2col --precision tf32 --out gpurun_out/alex 2>&1 | tail -2
head -12 gpurun_out/alex/sim_alexnet_b64_convgemm_tf32.csv
head -12 gpurun_out/alex/sim_alexnet_b64_convgemm_auto.csv
