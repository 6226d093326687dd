set -x
export HS_WATCHDOG_MS=5000
timeout 600 python -m pytest tests/test_gpu_wave.py -q -x 2>&1 | tail -5 > gpurun_out/pytest_wave.log
python tools/trace_wave.py c3 > gpurun_out/trace_wave_c3.txt 2>&1
for v in 1 0; do HS_WAVE_2SM=$v timeout 300 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('2sm $v', d['value'], d['roofline']['kernel_ms_per_forward'], d['plan'], d['e2e']['value'], d['clocks'])"; done > gpurun_out/wave_2sm.txt 2>&1
for lag in 2 3 4 6; do HS_WAVE_LAG=$lag timeout 300 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lag $lag', d['value'], d['roofline']['kernel_ms_per_forward'])"; done >> gpurun_out/wave_2sm.txt 2>&1
cat gpurun_out/pytest_wave.log gpurun_out/trace_wave_c3.txt; grep "2sm\|lag" gpurun_out/wave_2sm.txt
