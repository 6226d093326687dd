# f32-mode K1 as two fp16 passes (x fp16, W_ih fp16 hi/lo row-scaled) instead of three bf16 passes:
# parity suite, golden max-abs, benches c2-c5
mkdir -p gpurun_out/r5i
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r5i/pytest_gpu.log
cat gpurun_out/r5i/pytest_gpu.log
timeout 600 python -m pytest tests/test_gpu_golden.py -q -s 2>&1 | grep -i "max\|abs\|pass\|fail" | head -20 > gpurun_out/r5i/golden.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r5i/bench_c2.log 2>&1
for c in c3 c4 c5; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 > gpurun_out/r5i/bench_$c.log 2>&1; done
for f in gpurun_out/r5i/bench_c*.log; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['roofline']['kernel_ms_per_forward'],3), round(d['roofline']['gemm_ms_per_forward'],3), round(d['ms_per_step'],3), round(d['e2e']['value'],1) if d.get('e2e') else None)" || tail -3 $f; done
cat gpurun_out/r5i/golden.log
