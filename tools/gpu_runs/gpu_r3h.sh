# W-streaming recurrence with the first chunks resident in TMEM (c4)
set -x
mkdir -p gpurun_out/r3h
export HS_WATCHDOG_MS=30000
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/r3h/pytest_gpu.log
timeout 300 python -m pytest tests/test_gpu_golden.py -q -s -k c4 2>&1 | grep -E "max-abs|passed|failed" > gpurun_out/r3h/golden.log
for w in 0 1; do HS_W_TMEM=$w timeout 600 python bench.py --config c4 --no-cpu-baseline --steps 5 > gpurun_out/r3h/c4_w$w.log 2>&1; done
for w in 0 1; do HS_W_TMEM=$w HS_FORCE_STREAM=1 timeout 300 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -2 >> gpurun_out/r3h/golden.log; done
cat gpurun_out/r3h/pytest_gpu.log gpurun_out/r3h/golden.log
for f in gpurun_out/r3h/c4*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['e2e']['value'],1), d['roofline']['kernel_ms_per_forward'])" || tail -3 $f; done
