# async output drain for request streams: host-io tests + golden request path + e2e A/B (c2, c5)
set -x
mkdir -p gpurun_out/r3a
export HS_WATCHDOG_MS=20000
timeout 600 python -m pytest tests/test_gpu_host_io.py tests/test_gpu_golden.py tests/test_gpu_serving.py tests/test_executor.py tests/test_gpu_cells.py -m gpu -q -x 2>&1 | tail -4 > gpurun_out/r3a/tests.log
for a in 0 1; do HS_ASYNC_OUT=$a timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/r3a/c2_a$a.log 2>&1; done
for a in 0 1; do HS_ASYNC_OUT=$a timeout 600 python bench.py --config c5 --no-cpu-baseline --steps 5 > gpurun_out/r3a/c5_a$a.log 2>&1; done
for a in 0 1; do HS_ASYNC_OUT=$a timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 20 > gpurun_out/r3a/c3_a$a.log 2>&1; done
cat gpurun_out/r3a/tests.log
for f in gpurun_out/r3a/c*_a*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), round(d['e2e']['single_request_p50_ms'],3))" || tail -3 $f; done
