# Round-2 evidence after W_hh-in-TMEM: benches c2..c5 + reference arm, launch lists, full captures (CSV on the box)
set -x
mkdir -p gpurun_out/r2y
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py > gpurun_out/r2y/bench_c2.log 2>&1
for c in c3 c4 c5; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 > gpurun_out/r2y/bench_$c.log 2>&1; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2y/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2y/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2y/b_ncu_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/r2y/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2y/b_ncu_c3.log 2>&1
for k in c2 c3; do
  rep=/tmp/ncu_$k
  case $k in
    c2) timeout 900 ncu --set full --clock-control none --import-source on -k regex:recur_tc2 -s 2 -c 1 -o $rep -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2y/ncu_$k.log 2>&1 ;;
    c3) timeout 900 ncu --set full --clock-control none --import-source on -k regex:wave_fused -s 1 -c 1 -o $rep -f python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2y/ncu_$k.log 2>&1 ;;
  esac
  ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/r2y/ncu_${k}_raw.csv 2>&1
  ncu -i $rep.ncu-rep --page details --csv > gpurun_out/r2y/ncu_${k}_details.csv 2>&1
done
tail -n 1 gpurun_out/r2y/bench_*.log | cut -c1-300
