set -x
mkdir -p gpurun_out/r3p
export HS_WATCHDOG_MS=30000
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_golden.py tests/test_gpu_parity.py tests/test_gpu_cells.py -q -x -s 2>&1 | grep -E "c4 |passed|failed|Error" | tail -3 > gpurun_out/r3p/tests.log
TRACE_S=2 timeout 300 python tools/trace_recur.py c4 2>&1 | tail -16 > gpurun_out/r3p/trace.log
for rep in 1 2; do timeout 600 python bench.py --config c4 --no-cpu-baseline --steps 5 > gpurun_out/r3p/c4_$rep.log 2>&1; done
cat gpurun_out/r3p/tests.log gpurun_out/r3p/trace.log
for f in gpurun_out/r3p/c4*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['kernel_ms_per_forward'],3))" || tail -3 $f; done
