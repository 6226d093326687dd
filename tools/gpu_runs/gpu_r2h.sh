set -x
export HS_WATCHDOG_MS=5000
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
HS_WAVE_2SM=0 python tools/trace_wave.py c3 > gpurun_out/trace_wave_c3.txt 2>&1
HS_WAVE=0 TRACE_S=4 HS_RECUR_TRACE=gpurun_out/t.bin python tools/trace_recur.py c3 > gpurun_out/trace_c3_s4.txt 2>&1
python tools/trace_recur2.py > gpurun_out/trace_c2.txt 2>&1
for c in c2 c3; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['roofline']['kernel_ms_per_forward'], d['plan'], d['e2e']['value'], d['clocks'])"; done > gpurun_out/bench_r2h.txt 2>&1
HS_WAVE_2SM=0 timeout 300 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3-1sm', d['value'], d['roofline']['kernel_ms_per_forward'], d['plan'], d['e2e']['value'])" >> gpurun_out/bench_r2h.txt 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/trace_wave_c3.txt gpurun_out/trace_c3_s4.txt gpurun_out/trace_c2.txt gpurun_out/bench_r2h.txt
