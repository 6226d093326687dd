set -x
mkdir -p gpurun_out/r3o
timeout 600 ncu --set full --clock-control none -k regex:gemm_xproj_persistent -s 2 -c 1 -o /tmp/k1 -f python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r3o/ncu.log 2>&1
ncu -i /tmp/k1.ncu-rep --page raw --csv > gpurun_out/r3o/k1_raw.csv 2>&1
ncu -i /tmp/k1.ncu-rep --page details --csv > gpurun_out/r3o/k1_details.csv 2>&1
