set -x
mkdir -p gpurun_out/r3c
for sl in 2 3; do for a in 0 1; do HS_STREAM_SLOTS=$sl HS_ASYNC_OUT=$a timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/r3c/c2_s${sl}_a${a}.log 2>&1; done; done
for sl in 2 3; do for a in 0 1; do HS_STREAM_SLOTS=$sl HS_ASYNC_OUT=$a timeout 600 python bench.py --config c5 --no-cpu-baseline --steps 5 > gpurun_out/r3c/c5_s${sl}_a${a}.log 2>&1; done; done
for f in gpurun_out/r3c/c*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), round(d['e2e']['ms_per_step'],4))" || tail -3 $f; done
