# W_hh in TMEM for the single-group kernel and the wave: full GPU suite + bench A/B c2/c3/c5-shard
set -x
mkdir -p gpurun_out/r2w
export HS_WATCHDOG_MS=20000
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r2w/pytest_gpu.log
timeout 300 python -m pytest tests/test_gpu_golden.py -q -s 2>&1 | grep -E "max-abs|passed|failed" > gpurun_out/r2w/golden.log
for w in 0 1; do
  HS_W_TMEM=$w timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/r2w/c2_w$w.log 2>&1
  HS_W_TMEM=$w timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 20 > gpurun_out/r2w/c3_w$w.log 2>&1
  HS_W_TMEM=$w timeout 300 python bench.py --config c5 --global-batch 32 --no-cpu-baseline --steps 5 > gpurun_out/r2w/c5s_w$w.log 2>&1
done
cat gpurun_out/r2w/pytest_gpu.log gpurun_out/r2w/golden.log
for f in gpurun_out/r2w/c*_w*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), d['roofline']['kernel_ms_per_forward'])" || tail -3 $f; done
