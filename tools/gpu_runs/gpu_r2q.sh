# c4 W ring depth A/B (4 vs 5 stages)
set -x
mkdir -p gpurun_out/r2q
for r in 4 5; do HS_W_RING=$r timeout 600 python bench.py --config c4 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r2q/c4_ring$r.log 2>&1; done
for f in gpurun_out/r2q/c4_ring*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['roofline']['kernel_ms_per_forward'])"; done
