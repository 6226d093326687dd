# Round-2 first GPU pass: new full-size golden + robustness tests, then the whole GPU tier and a c2 bench.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_robust.py -v -s -x 2>&1 | tail -60 > gpurun_out/pytest_r2a.log
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.log 2>&1
tail -n 40 gpurun_out/pytest_r2a.log gpurun_out/pytest_gpu.log; tail -c 3000 gpurun_out/bench_c2.log
