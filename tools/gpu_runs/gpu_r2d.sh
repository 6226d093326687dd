set -x
python tools/trace_wave.py c3 > gpurun_out/trace_wave_c3.txt 2>&1
HS_WAVE=0 HS_RECUR_TRACE=gpurun_out/trace_c3_layer.bin TRACE_S=4 python tools/trace_recur.py c3 > gpurun_out/trace_c3_layer.txt 2>&1
for lag in 3 4 5 6; do HS_WAVE_LAG=$lag timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lag $lag', d['value'], d['roofline']['kernel_ms_per_forward'], d['clocks'])"; done > gpurun_out/wave_lag.txt 2>&1
cat gpurun_out/trace_wave_c3.txt gpurun_out/trace_c3_layer.txt; grep lag gpurun_out/wave_lag.txt
