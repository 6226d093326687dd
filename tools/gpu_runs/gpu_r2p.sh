# hybrid model check after the crossing-latency / host-cell changes; launch lists c2/c3/c4 for profiles
set -x
mkdir -p gpurun_out/r2p
timeout 900 python tools/hybrid_model_check.py c1 gpurun_out/r2p/hybrid_c1.json > gpurun_out/r2p/hybrid_c1.log 2>&1
timeout 1500 python tools/hybrid_model_check.py c3 gpurun_out/r2p/hybrid_c3.json --seq 64 > gpurun_out/r2p/hybrid_c3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_cells.py tests/test_executor.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/r2p/pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2p/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2p/b_ncu_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/r2p/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2p/b_ncu_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2p/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2p/b_ncu_c4.log 2>&1
cat gpurun_out/r2p/pytest.log
