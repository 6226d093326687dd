# pytest -m gpu, c2 bench, ncu launch list + recurrence full capture
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:recur_tc -s 2 -c 1 -o gpurun_out/recur_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_recur.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/ncu_recur.log
