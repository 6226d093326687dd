# Round-2 ncu evidence (launch lists + full captures of the dominant kernels) and the serving study.
set -x
export HS_WATCHDOG_MS=60000
mkdir -p gpurun_out/r2m
timeout 600 python -m pytest tests/test_gpu_serving.py -q -x 2>&1 | tail -15 > gpurun_out/r2m/pytest_serving.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2m/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2m/b_ncu_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/r2m/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2m/b_ncu_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2m/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2m/b_ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:recur_tc2 -s 2 -c 1 -o gpurun_out/r2m/c2_recur_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2m/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wave_fused -s 1 -c 1 -o gpurun_out/r2m/c3_wave_full -f python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2m/ncu_c3.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:recur_tc_kernel -s 8 -c 1 -o gpurun_out/r2m/c4_recur_full -f python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2m/ncu_c4.log 2>&1
timeout 1200 python tools/serving_report.py gpurun_out/r2m/serving.json > gpurun_out/r2m/serving.log 2>&1
tail -n 3 gpurun_out/r2m/*.log
