for W in 170 300 600 1000; do echo "== waste_pct $W"; python tools/fuzz_perf.py --tune "{\"waste_pct\": $W}" 2>&1 | sort -k2 -n -r | head -40 | grep -E " on 7x7 b=64| on 20x20 b=50| 28x28 b=16 s=1 p=3|96x3x3x256 on 12x12" ; done
timeout 600 python -m pytest tests/test_fuzz_gpu.py -q -m gpu 2>&1 | tail -2
