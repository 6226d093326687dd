# one TMA per step for the K-slice (two-group kernel): parity + trace + A/B
set -x
mkdir -p gpurun_out/r2x
export HS_WATCHDOG_MS=20000
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_golden.py tests/test_gpu_parity.py -q -x -s 2>&1 | grep -E "max-abs|passed|failed|Error" | head -12 > gpurun_out/r2x/tests.log
timeout 300 python tools/trace_recur2.py > gpurun_out/r2x/trace.log 2>&1
for h in 0 1; do HS_H_TMA1=$h timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/r2x/c2_h$h.log 2>&1; done
for h in 0 1; do HS_H_TMA1=$h timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/r2x/c2b_h$h.log 2>&1; done
cat gpurun_out/r2x/tests.log gpurun_out/r2x/trace.log
for f in gpurun_out/r2x/c2*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), d['roofline']['kernel_ms_per_forward'])" || tail -3 $f; done
