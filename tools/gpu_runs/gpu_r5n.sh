# hidden layers K1 as two fp16 passes (layer 0 keeps three bf16 products), fused K-blocks in every K1 kernel:
# A/B benches (HS_K1_F16_HIDDEN=0/1) c2 x2, c3, c4
mkdir -p gpurun_out/r5n
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/r5n/pytest_gpu.log
cat gpurun_out/r5n/pytest_gpu.log
timeout 600 python -m pytest tests/test_gpu_golden.py -q -s 2>&1 | grep "max-abs" | cut -c1-60,200-400 > gpurun_out/r5n/golden.log
cat gpurun_out/r5n/golden.log
for i in 1 2; do for v in 1 0; do HS_K1_F16_HIDDEN=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r5n/c2_h${v}_$i.log 2>&1; done; done
for v in 1 0; do HS_K1_F16_HIDDEN=$v timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/r5n/c3_h$v.log 2>&1; done
for v in 1 0; do HS_K1_F16_HIDDEN=$v timeout 900 python bench.py --config c4 --no-cpu-baseline --steps 5 > gpurun_out/r5n/c4_h$v.log 2>&1; done
for f in gpurun_out/r5n/c*_h*.log; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['roofline']['kernel_ms_per_forward'],3), round(d['roofline']['gemm_ms_per_forward'],3), round(d['ms_per_step'],4), round(d['e2e']['value'],1))" 2>/dev/null || tail -2 $f; done
