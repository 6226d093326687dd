# Round-2 evidence: ncu launch list (c2) + full captures (c2 recurrence, c3 wave, c4 W-streaming
# recurrence), compute-sanitizer on the production kernel families.
set -x
export HS_WATCHDOG_MS=60000
mkdir -p gpurun_out/r2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2/b_ncu_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/r2/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2/b_ncu_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:recur_tc2 -s 2 -c 1 -o gpurun_out/r2/c2_recur_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wave_fused -s 1 -c 1 -o gpurun_out/r2/c3_wave_full -f python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2/ncu_c3.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:recur_tc_kernel -s 8 -c 1 -o gpurun_out/r2/c4_recur_full -f python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2/ncu_c4.log 2>&1
for tool in racecheck synccheck memcheck; do timeout 900 compute-sanitizer --tool $tool python tools/sanitize_prod.py > gpurun_out/r2/$tool.log 2>&1; done
tail -n 4 gpurun_out/r2/*.log
ls -la gpurun_out/r2
