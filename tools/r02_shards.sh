#!/bin/bash
# The strong-scaling shards (b = 64, 32, 16 of the global 128) timed alone on one GPU.
mkdir -p gpurun_out/shards
for N in 2 4 8; do
  python bench.py --shard-of $N --steps 20 --warmup 5 --quick --no-cpu-baseline > gpurun_out/shards/shard_of_$N.json 2> gpurun_out/shards/err_$N.log
  python -c "import json; d=json.loads(open('gpurun_out/shards/shard_of_$N.json').read().strip().splitlines()[-1]); print('shard of $N: b', d['config']['batch_per_gpu'], 'step us', round(d['ms_per_step']*1e3,1), [ (l['layer'][8:], round(l['ms']*1e3,1)) for l in d['roofline']['per_layer']], 'launches', d['gpu_launches'])"
done
