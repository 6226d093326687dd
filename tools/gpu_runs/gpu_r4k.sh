# c5: two-group slices of 128 rows (8 cells per thread, HS_TWO_GROUP_CELLS=8 build) vs slices of 64 (default)
mkdir -p gpurun_out/r4k
C8=paper_2307_11339_b200/_lib/libhsrnn_c8.so
for i in 1 2; do
  unset HS_LIB_PATH; timeout 600 python bench.py --config c5 --no-cpu-baseline --steps 5 > gpurun_out/r4k/c5_base_$i.log 2>&1
  HS_LIB_PATH=$C8 timeout 600 python bench.py --config c5 --no-cpu-baseline --steps 5 > gpurun_out/r4k/c5_c8_$i.log 2>&1
done
HS_LIB_PATH=$C8 timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r4k/c2_c8.log 2>&1
HS_LIB_PATH=$C8 timeout 900 python -m pytest tests/test_gpu_random_shapes.py tests/test_gpu_golden.py tests/test_gpu_tc.py tests/test_gpu_graph.py -q -x 2>&1 | tail -3 > gpurun_out/r4k/pytest_c8.log
for f in gpurun_out/r4k/c*_*.log; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['roofline']['kernel_ms_per_forward'],3), d['plan'].get('batch_slices'), round(d['e2e']['value'],1) if d.get('e2e') else None)"; done
cat gpurun_out/r4k/pytest_c8.log
