# MMA issuer: TMEM chunks waited for up front, MMAs back to back (new) vs interleaved (base build): c4/c2/c3/c5 A/B, parity sweep
mkdir -p gpurun_out/r4i
B=paper_2307_11339_b200/_lib/libhsrnn_base.so
for i in 1 2; do
  for v in base new; do
    if [ $v = base ]; then export HS_LIB_PATH=$B; else unset HS_LIB_PATH; fi
    timeout 600 python bench.py --config c4 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r4i/c4_${v}_$i.log 2>&1
    timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r4i/c2_${v}_$i.log 2>&1
    timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/r4i/c3_${v}_$i.log 2>&1
  done
done
for v in base new; do
  if [ $v = base ]; then export HS_LIB_PATH=$B; else unset HS_LIB_PATH; fi
  timeout 600 python bench.py --config c5 --no-cpu-baseline --steps 5 > gpurun_out/r4i/c5_${v}.log 2>&1
done
unset HS_LIB_PATH
timeout 900 python -m pytest tests/test_gpu_random_shapes.py tests/test_gpu_golden.py tests/test_gpu_tc.py -q -x 2>&1 | tail -3 > gpurun_out/r4i/pytest.log
for f in gpurun_out/r4i/c*_*.log; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['roofline']['kernel_ms_per_forward'],3), round(d['e2e']['value'],1) if d.get('e2e') else None)"; done
cat gpurun_out/r4i/pytest.log
