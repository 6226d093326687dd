# two TMEM accumulators (HS_NACC=2) vs one: c4 / c2 / c5 A/B, c4 trace, parity sweep
mkdir -p gpurun_out/r4c
for i in 1 2; do
  for n in 1 2; do
    HS_NACC=$n timeout 600 python bench.py --config c4 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r4c/c4_nacc${n}_$i.log 2>&1
    HS_NACC=$n timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r4c/c2_nacc${n}_$i.log 2>&1
  done
done
for n in 1 2; do HS_NACC=$n timeout 600 python bench.py --config c5 --no-cpu-baseline --steps 5 > gpurun_out/r4c/c5_nacc${n}.log 2>&1; done
HS_NACC=2 TRACE_S=2 timeout 600 python tools/trace_recur.py c4 /tmp/tr_c4.bin > gpurun_out/r4c/trace_c4_nacc2.txt 2>&1
HS_NACC=2 timeout 900 python -m pytest tests/test_gpu_random_shapes.py tests/test_gpu_golden.py tests/test_gpu_tc.py -q -x 2>&1 | tail -3 > gpurun_out/r4c/pytest_nacc2.log
for f in gpurun_out/r4c/c*_nacc*.log; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['roofline']['kernel_ms_per_forward'], d['e2e']['value'] if d.get('e2e') else None)"; done
cat gpurun_out/r4c/trace_c4_nacc2.txt gpurun_out/r4c/pytest_nacc2.log
