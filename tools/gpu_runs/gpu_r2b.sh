# Round-2: layer wavefront parity + c3/c2 bench
set -x
export HS_WATCHDOG_MS=5000
timeout 600 python -m pytest tests/test_gpu_wave.py -v -s -x 2>&1 | tail -40 > gpurun_out/pytest_wave.log
timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
HS_WAVE=0 timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3_nowave.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
tail -n 40 gpurun_out/pytest_wave.log; tail -c 1500 gpurun_out/bench_c3.log; tail -c 600 gpurun_out/bench_c3_nowave.log; tail -5 gpurun_out/pytest_gpu.log
