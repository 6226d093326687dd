set -x
mkdir -p gpurun_out/r3b
for rep in 1 2; do for a in 0 1; do HS_ASYNC_OUT=$a timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/r3b/c2_a${a}_$rep.log 2>&1; done; done
for f in gpurun_out/r3b/c2_a*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), round(d['e2e']['ms_per_step'],4))" || tail -3 $f; done
