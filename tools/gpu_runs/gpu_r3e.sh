# TMEM-resident W_hh plan mode (c5: 3 unstreamed batch slices instead of 4 streamed)
set -x
mkdir -p gpurun_out/r3e
export HS_WATCHDOG_MS=30000
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_golden.py tests/test_gpu_parity.py tests/test_gpu_host_io.py -q -x -s 2>&1 | grep -E "max-abs|passed|failed|Error" | tail -14 > gpurun_out/r3e/tests.log
timeout 900 python bench.py --config c5 --no-cpu-baseline --steps 5 > gpurun_out/r3e/c5.log 2>&1
HS_FORCE_STREAM=1 timeout 900 python bench.py --config c5 --no-cpu-baseline --steps 5 > gpurun_out/r3e/c5_stream.log 2>&1
cat gpurun_out/r3e/tests.log
for f in gpurun_out/r3e/c5*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), d['roofline']['kernel_ms_per_forward'], d['roofline']['gemm_ms_per_forward'], d['plan'])" || tail -3 $f; done
