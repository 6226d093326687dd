set -x
mkdir -p gpurun_out/r3f
export HS_WATCHDOG_MS=30000
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_golden.py -q -x -s 2>&1 | grep -E "c5|passed|failed|Error" | tail -6 > gpurun_out/r3f/tests.log
for w in 1 0; do HS_W_TMEM=$w timeout 900 python bench.py --config c5 --no-cpu-baseline --steps 5 > gpurun_out/r3f/c5_w$w.log 2>&1; done
cat gpurun_out/r3f/tests.log
for f in gpurun_out/r3f/c5*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), d['roofline']['kernel_ms_per_forward'], d['plan'])" || tail -3 $f; done
