set -x
mkdir -p gpurun_out/r3r
for lag in 1 2 3 4 6; do HS_WAVE_LAG=$lag timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 20 > gpurun_out/r3r/c3_lag$lag.log 2>&1; done
for f in gpurun_out/r3r/c3_*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), round(d['roofline']['kernel_ms_per_forward'],4))" || tail -3 $f; done
