python bench.py --steps 20 --warmup 5 --quick --no-cpu-baseline --concurrent 1,2,3,4,7 > gpurun_out/conc_b128.json 2> gpurun_out/conc_b128.err
python bench.py --steps 20 --warmup 5 --quick --no-cpu-baseline --concurrent 1,2,3,4,7 --shard-of 8 > gpurun_out/conc_b16.json 2> gpurun_out/conc_b16.err
python - <<'PY'
import json
for f in ("gpurun_out/conc_b128.json","gpurun_out/conc_b16.json"):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], {k:(round(v["ms_per_step"],4), round(v["tf32_frac"],3), v.get("parity_pass")) for k,v in d["concurrent"]["streams"].items()})
    except Exception as e: print(f, "ERR", e)
PY
tail -3 gpurun_out/conc_b128.err
