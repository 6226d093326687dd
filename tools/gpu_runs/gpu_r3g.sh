# two-group recurrence for batch slices (TMEM W where needed): c5
set -x
mkdir -p gpurun_out/r3g
export HS_WATCHDOG_MS=30000
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_golden.py tests/test_gpu_parity.py -q -x -s 2>&1 | grep -E "c5|sliced|passed|failed|Error" | tail -8 > gpurun_out/r3g/tests.log
for t in 1 0; do HS_TWO_GROUPS=$t timeout 900 python bench.py --config c5 --no-cpu-baseline --steps 5 > gpurun_out/r3g/c5_two$t.log 2>&1; done
timeout 900 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/r3g/c2.log 2>&1
cat gpurun_out/r3g/tests.log
for f in gpurun_out/r3g/c*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), d['roofline']['kernel_ms_per_forward'])" || tail -3 $f; done
