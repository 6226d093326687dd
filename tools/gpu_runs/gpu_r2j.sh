set -x
export HS_WATCHDOG_MS=5000
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/pytest_gpu.log
python tools/trace_wave.py c3 > gpurun_out/trace_wave_c3.txt 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/trace_wave_c3.txt
