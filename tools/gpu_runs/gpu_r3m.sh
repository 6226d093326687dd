set -x
mkdir -p gpurun_out/r3m
export HS_WATCHDOG_MS=20000
timeout 600 python -m pytest tests/test_gpu_host_io.py tests/test_gpu_golden.py -q -x 2>&1 | tail -2 > gpurun_out/r3m/tests.log
timeout 300 python tools/timeline_host.py c2 2>/dev/null | tail -22 > gpurun_out/r3m/timeline.log
for rep in 1 2; do for v in 1 2; do HS_DRAIN_STREAMS=$v timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/r3m/c2_s${v}_$rep.log 2>&1; done; done
for v in 1 2; do HS_DRAIN_STREAMS=$v timeout 600 python bench.py --config c5 --no-cpu-baseline --steps 5 > gpurun_out/r3m/c5_s$v.log 2>&1; done
cat gpurun_out/r3m/tests.log gpurun_out/r3m/timeline.log
for f in gpurun_out/r3m/c*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), round(d['e2e']['single_request_p50_ms'],3))" || tail -3 $f; done
