# W_hh in TMEM (two-group kernel): parity + trace + bench A/B
set -x
mkdir -p gpurun_out/r2v
export HS_WATCHDOG_MS=20000
timeout 300 python -m pytest tests/test_gpu_golden.py -q -s -k "c2" 2>&1 | grep -E "max-abs|passed|failed|Error" | head -5 > gpurun_out/r2v/golden.log
timeout 300 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -3 >> gpurun_out/r2v/golden.log
timeout 300 python tools/trace_recur2.py > gpurun_out/r2v/trace.log 2>&1
for w in 0 1; do HS_W_TMEM=$w timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/r2v/bench_w$w.log 2>&1; done
cat gpurun_out/r2v/golden.log gpurun_out/r2v/trace.log
for w in 0 1; do python -c "import json; d=json.loads(open('gpurun_out/r2v/bench_w$w.log').read().strip().splitlines()[-1]); print('w_tmem=$w', d['value'], d['roofline']['kernel_ms_per_forward'])" || tail -3 gpurun_out/r2v/bench_w$w.log; done
