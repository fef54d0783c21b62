#!/bin/bash
# Round-2: explicit path (K1 slab im2col + K2 TMA-fed GEMM) and fc GEMM: parity, then timings.
timeout 900 python -m pytest tests/test_explicit_path_gpu.py tests/test_simulator.py tests/test_reference_surface_gpu.py -x -q -m gpu > gpurun_out/explicit_tests.log 2>&1
echo "explicit tests rc=$?"; tail -15 gpurun_out/explicit_tests.log
timeout 600 python tools/time_explicit.py > gpurun_out/explicit_times.log 2>&1; echo "times rc=$?"; cat gpurun_out/explicit_times.log
