set -x
mkdir -p gpurun_out/r2u
timeout 900 python -m pytest tests/test_gpu_golden.py -q -s 2>&1 | grep -E "max-abs|passed|failed" > gpurun_out/r2u/golden.log
timeout 600 python bench.py > gpurun_out/r2u/bench_c2.log 2>&1
timeout 600 python bench.py --config c3 --no-cpu-baseline --steps 10 > gpurun_out/r2u/bench_c3.log 2>&1
cat gpurun_out/r2u/golden.log
