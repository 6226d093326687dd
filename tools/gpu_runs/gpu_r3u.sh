set -x
mkdir -p gpurun_out/r3u
for t in 0 1; do HS_TWO_GROUPS=$t timeout 600 python bench.py --config c5 --global-batch 32 --no-cpu-baseline --steps 5 > gpurun_out/r3u/c5s_two$t.log 2>&1; done
for t in 0 1; do HS_TWO_GROUPS=$t timeout 600 python bench.py --config c3 --no-cpu-baseline --steps 20 > gpurun_out/r3u/c3_two$t.log 2>&1; done
for f in gpurun_out/r3u/*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), round(d['roofline']['kernel_ms_per_forward'],3), d['plan']['layer_wave'])" || tail -2 $f; done
