# c4 W ring 4 vs 5 with the TMEM-resident chunks (A/B, alternating, one box)
set -x
mkdir -p gpurun_out/r4a
for i in 1 2; do
  for r in 4 5; do
    HS_W_RING=$r timeout 600 python bench.py --config c4 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r4a/c4_ring${r}_$i.log 2>&1
  done
done
HS_W_RING=5 timeout 900 python -m pytest tests/test_gpu_random_shapes.py tests/test_gpu_golden.py -q -x 2>&1 | tail -3 > gpurun_out/r4a/pytest_ring5.log
for f in gpurun_out/r4a/c4_ring*.log; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['roofline']['kernel_ms_per_forward'])"; done
cat gpurun_out/r4a/pytest_ring5.log
