set -x
mkdir -p gpurun_out/r3i
HS_FORCE_STREAM=1 timeout 300 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | grep -E "Error|FAILED|assert" | head -5 > gpurun_out/r3i/forced.log
for rep in 1 2; do for w in 0 1; do HS_W_TMEM=$w timeout 600 python bench.py --config c4 --no-cpu-baseline --steps 5 > gpurun_out/r3i/c4_w${w}_$rep.log 2>&1; done; done
cat gpurun_out/r3i/forced.log
for f in gpurun_out/r3i/c4*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['e2e']['value'],1), d['roofline']['kernel_ms_per_forward'])" || tail -3 $f; done
