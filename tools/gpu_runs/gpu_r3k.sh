# Round-2 evidence at the current state: GPU suite, smoke, benches c2..c5 + reference arm + c4 pipeline N=1 +
# c5 8-way shard size, launch lists (c2, c4), ncu full captures exported to CSV (c2, c4), peaks probe
set -x
mkdir -p gpurun_out/r3k
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/r3k/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3k/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r3k/bench_c2.log 2>&1
for c in c3 c4 c5; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 > gpurun_out/r3k/bench_$c.log 2>&1; done
timeout 600 python bench.py --config c5 --global-batch 32 --no-cpu-baseline --steps 5 > gpurun_out/r3k/bench_c5_shard32.log 2>&1
timeout 600 python bench.py --config c4 --mode pipeline --steps 3 --warmup 3 > gpurun_out/r3k/bench_c4_pipeline.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r3k/bench_ref.log 2>&1
timeout 300 python tools/peak_probe.py gpurun_out/r3k/peaks.json > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r3k/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r3k/b_ncu_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r3k/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r3k/b_ncu_c4.log 2>&1
for k in c2 c4; do
  rep=/tmp/ncu_$k
  case $k in
    c2) timeout 900 ncu --set full --clock-control none --import-source on -k regex:recur_tc2 -s 2 -c 1 -o $rep -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r3k/ncu_$k.log 2>&1 ;;
    c4) timeout 1200 ncu --set full --clock-control none --import-source on -k regex:recur_tc_kernel -s 8 -c 1 -o $rep -f python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r3k/ncu_$k.log 2>&1 ;;
  esac
  ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/r3k/ncu_${k}_raw.csv 2>&1
  ncu -i $rep.ncu-rep --page details --csv > gpurun_out/r3k/ncu_${k}_details.csv 2>&1
done
cat gpurun_out/r3k/pytest_gpu.log gpurun_out/r3k/smoke.log
