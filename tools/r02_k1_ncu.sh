mkdir -p gpurun_out/r02x
python tools/ncu_cases.py explicit > /dev/null 2>&1 && ncu --set full --cache-control all --clock-control none --import-source on -k regex:"im2col" -s 1 -c 1 -o gpurun_out/r02x/k1 python tools/ncu_cases.py explicit > gpurun_out/r02x/ncu_k1.log 2>&1
python tools/ncu_summary.py gpurun_out/r02x/k1.ncu-rep > gpurun_out/r02x/k1_raw.txt 2>&1
python tools/ncu_stalls.py gpurun_out/r02x/k1.ncu-rep 40 > gpurun_out/r02x/k1_hot.txt 2>&1
