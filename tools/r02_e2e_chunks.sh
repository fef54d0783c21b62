for kb in ${KBS:-8192 16384 32768 65536}; do
  python bench.py --steps 5 --warmup 3 --quick --no-cpu-baseline --no-parity --tune "{\"host_chunk_kb\":$kb}" > gpurun_out/e2e_$kb.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/e2e_$kb.json').read().strip().splitlines()[-1]); print('chunk_kb $kb e2e GFLOPS', round(d['e2e']['value']), 'ms', round(d['e2e']['ms_per_step'],3))"
done
