mkdir -p gpurun_out/r02p
CMD="python bench.py --steps 2 --warmup 3 --quick --no-cpu-baseline --no-parity"
K='regex:sw_conv|splitk'
for T in '{"sk":0}' '{"sk":0,"pdl":0}' '{"splitk":-1,"sk":0,"tail":0}'; do
  n=$(echo $T | tr -cd 'a-z0-9')
  ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 60 --csv --log-file gpurun_out/r02p/l_$n.csv $CMD --tune "$T" > gpurun_out/r02p/ncu_$n.log 2>&1
  echo "tune $T rc=$? launches=$(grep -c sw_conv gpurun_out/r02p/l_$n.csv)"
done
ncu --graph-profiling graph --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02p/l_graph.csv $CMD > gpurun_out/r02p/ncu_graph.log 2>&1
echo "graph-profiling graph rc=$?"; tail -4 gpurun_out/r02p/l_graph.csv | cut -c1-250
for L in r50_3x3_56_64 r50_3x3_14_256 r50_3x3_7_512 r50_3x3_s2_56_128; do
  echo "== $L"; CGB_DEBUG_SW=64 timeout 60 python tools/run_layer.py --layer $L --reps 10 2>&1 | tail -9
done
