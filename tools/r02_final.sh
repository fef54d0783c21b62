#!/bin/bash
# Round-end recheck: the driver's sequence on one box (GPU tests, smoke, both bench arms).
mkdir -p gpurun_out/final
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/final/gpu_tests.txt 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/final/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/final/smoke.txt
timeout 900 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err; echo "reference arm rc=$?"; tail -c 400 gpurun_out/final/bench_reference.json
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final/bench_steps20.json 2> gpurun_out/final/bench_steps20.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/final/bench_steps20.json').read().strip().splitlines()[-1]); print('step ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']), 'parity', d['parity']['tf32']['pass'], d['clocks'])"
