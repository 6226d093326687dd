# A/B: L2 eviction policies on the W-streaming recurrence (HS_L2_HINTS bits: 1 W evict_last, 2 xproj/y evict_first)
set -x
mkdir -p gpurun_out/r2l
for c in c4 c5; do for h in 0 1 3; do
  HS_L2_HINTS=$h timeout 600 python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r2l/b_${c}_h$h.log 2>&1
done; done
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r2l/pytest.log
for f in gpurun_out/r2l/b_*.log; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_forward'])"; done
cat gpurun_out/r2l/pytest.log
