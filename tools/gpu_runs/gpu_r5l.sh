# K1 fused three-product K-blocks (one load of X_hi/X_lo/W_hi/W_lo per K-block) vs pass-major (HS_K1_FUSED3=0):
# parity first (K1-heavy tests), then A/B benches c2/c3/c4 x2, then ncu of the K1 head
mkdir -p gpurun_out/r5l
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_cells.py tests/test_gpu_wave.py -q -x 2>&1 | tail -3 > gpurun_out/r5l/pytest.log
cat gpurun_out/r5l/pytest.log
for i in 1 2; do
  for v in 1 0; do
    HS_K1_FUSED3=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r5l/c2_f${v}_${i}b.log 2>&1
    HS_K1_FUSED3=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r5l/c2_f${v}_$i.log 2>&1
    HS_K1_FUSED3=$v timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/r5l/c3_f${v}_$i.log 2>&1
  done
done
for v in 1 0; do HS_K1_FUSED3=$v timeout 900 python bench.py --config c4 --no-cpu-baseline --steps 5 > gpurun_out/r5l/c4_f${v}.log 2>&1; done
for f in gpurun_out/r5l/c*_f*.log; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['roofline']['kernel_ms_per_forward'],3), round(d['roofline']['gemm_ms_per_forward'],3), round(d['ms_per_step'],4), round(d['e2e']['value'],1))" 2>/dev/null; done
for v in 1 0; do HS_K1_FUSED3=$v timeout 600 ncu --set full --clock-control none -k regex:gemm_xproj_persistent -s 2 -c 1 -o /tmp/k1_f$v -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; ncu -i /tmp/k1_f$v.ncu-rep --page raw --csv > gpurun_out/r5l/ncu_k1_f${v}_raw.csv 2>&1; done
