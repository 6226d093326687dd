# Round 2: cell-level entry points (TC segments, profile_cells), serving study, hybrid model check,
# full GPU suite; ncu summaries exported to CSV on the box (the .ncu-rep files stay there).
set -x
export HS_WATCHDOG_MS=60000
mkdir -p gpurun_out/r2n
timeout 900 python -m pytest tests/test_gpu_cells.py -q -x 2>&1 | tail -25 > gpurun_out/r2n/pytest_cells.log
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -25 > gpurun_out/r2n/pytest_gpu.log
timeout 900 python tools/hybrid_model_check.py c1 gpurun_out/r2n/hybrid_c1.json > gpurun_out/r2n/hybrid_c1.log 2>&1
timeout 1500 python tools/hybrid_model_check.py c3 gpurun_out/r2n/hybrid_c3.json --seq 64 > gpurun_out/r2n/hybrid_c3.log 2>&1
timeout 1500 python tools/serving_report.py gpurun_out/r2n/serving.json > gpurun_out/r2n/serving.log 2>&1
for k in c2 c3 c4; do
  rep=/tmp/ncu_$k
  case $k in
    c2) timeout 900 ncu --set full --clock-control none --import-source on -k regex:recur_tc2 -s 2 -c 1 -o $rep -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2n/ncu_$k.log 2>&1 ;;
    c3) timeout 900 ncu --set full --clock-control none --import-source on -k regex:wave_fused -s 1 -c 1 -o $rep -f python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2n/ncu_$k.log 2>&1 ;;
    c4) timeout 1200 ncu --set full --clock-control none --import-source on -k regex:recur_tc_kernel -s 8 -c 1 -o $rep -f python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2n/ncu_$k.log 2>&1 ;;
  esac
  ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/r2n/ncu_${k}_raw.csv 2>&1
  ncu -i $rep.ncu-rep --page details --csv > gpurun_out/r2n/ncu_${k}_details.csv 2>&1
  ncu -i $rep.ncu-rep --page source --csv > gpurun_out/r2n/ncu_${k}_source.csv 2>&1
done
ls -la gpurun_out/r2n
tail -n 4 gpurun_out/r2n/*.log
