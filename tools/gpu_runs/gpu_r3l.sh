set -x
mkdir -p gpurun_out/r3l
export HS_WATCHDOG_MS=20000
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_golden.py tests/test_gpu_host_io.py -q -x -s 2>&1 | grep -E "c2 |passed|failed|Error" | tail -4 > gpurun_out/r3l/tests.log
timeout 300 python tools/trace_recur2.py > gpurun_out/r3l/trace.log 2>&1
for rep in 1 2; do for v in 0 1; do HS_H_VEC=$v timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/r3l/c2_v${v}_$rep.log 2>&1; done; done
cat gpurun_out/r3l/tests.log gpurun_out/r3l/trace.log
for f in gpurun_out/r3l/c2_*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), round(d['roofline']['kernel_ms_per_forward'],4))" || tail -3 $f; done
