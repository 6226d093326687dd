set -x
export HS_WATCHDOG_MS=5000
timeout 300 python -m pytest "tests/test_gpu_wave.py::test_wave_matches_oracle" -q -x 2>&1 | grep -i "error\|passed\|failed" | head -20 > gpurun_out/pytest_wave.log
for cap in 4 8 20; do HS_WAVE_2SM=0 HS_WAVE_K1_CTAS=$cap python tools/trace_wave.py c3 2>&1 | head -6; done > gpurun_out/trace_cap.txt
for cap in 4 8 20 40; do HS_WAVE_K1_CTAS=$cap python tools/trace_wave.py c3 2>&1 | head -6; done > gpurun_out/trace_cap2.txt
cat gpurun_out/pytest_wave.log gpurun_out/trace_cap.txt gpurun_out/trace_cap2.txt
