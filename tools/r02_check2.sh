timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_fullsize.py -x -q -m gpu > gpurun_out/tests2.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/tests2.log
timeout 600 python bench.py --steps 20 --warmup 5 --quick --no-cpu-baseline > gpurun_out/bench2.log 2>&1; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench2.log').read().strip().splitlines()[-1]); print('step ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4), [ (l['layer'][8:], l['ms']) for l in d['roofline']['per_layer']], d['clocks'])"
python tools/bench_configs.py --configs C3,C4,C5 --out gpurun_out/configs2.json > gpurun_out/configs2.log 2>&1; tail -1 gpurun_out/configs2.log | cut -c1-900
