set -x
mkdir -p gpurun_out/r3v
export HS_WATCHDOG_MS=30000
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r3v/pytest.log
timeout 300 python -m pytest tests/test_gpu_golden.py -q -s -k c5 2>&1 | grep -E "max-abs" > gpurun_out/r3v/golden.log
timeout 600 python bench.py --config c5 --global-batch 32 --no-cpu-baseline --steps 5 > gpurun_out/r3v/c5s.log 2>&1
cat gpurun_out/r3v/pytest.log gpurun_out/r3v/golden.log
python -c "import json; d=json.loads(open('gpurun_out/r3v/c5s.log').read().strip().splitlines()[-1]); print(round(d['value']), round(d['e2e']['value']))"
