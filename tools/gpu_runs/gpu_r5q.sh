# c3 layer-wave lag (M-tiles) after the lighter hidden-layer K1: 2 vs 3 (default) vs 4
mkdir -p gpurun_out/r5q
for i in 1 2; do for lag in 2 3 4; do HS_WAVE_LAG=$lag timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/r5q/c3_lag${lag}_$i.log 2>&1; done; done
for f in gpurun_out/r5q/*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['roofline']['kernel_ms_per_forward'],3), round(d['e2e']['value'],1))"; done
