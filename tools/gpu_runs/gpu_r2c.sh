# wave diagnostics: trace, lag sweep, layer-0 K1 before the wave
set -x
python tools/trace_wave.py c3 > gpurun_out/trace_wave_c3.txt 2>&1
for lag in 1 2 4 8; do HS_WAVE_LAG=$lag timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lag $lag', d['value'], d['roofline']['kernel_ms_per_forward'], d['clocks'])"; done > gpurun_out/wave_lag.txt 2>&1
HS_WAVE_K1L0=1 timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c3_k1l0.log
cat gpurun_out/trace_wave_c3.txt gpurun_out/wave_lag.txt; tail -c 300 gpurun_out/bench_c3_k1l0.log
