# 256x256 super-tile persistent K1: parity + A/B (c5, c2) + ncu of the new kernel
set -x
mkdir -p gpurun_out/r3t
export HS_WATCHDOG_MS=30000
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r3t/pytest.log
for rep in 1 2; do for v in 0 1; do HS_GEMM_ST2=$v timeout 600 python bench.py --config c5 --no-cpu-baseline --steps 5 > gpurun_out/r3t/c5_st$v_$rep.log 2>&1; HS_GEMM_ST2=$v timeout 600 python bench.py --config c5 --no-cpu-baseline --steps 5 > gpurun_out/r3t/c5_st${v}_$rep.log 2>&1; done; done
for v in 0 1; do HS_GEMM_ST2=$v timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/r3t/c2_st$v.log 2>&1; done
timeout 600 ncu --set full --clock-control none -k regex:gemm_xproj_persistent2 -s 2 -c 1 -o /tmp/k1b -f python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r3t/ncu.log 2>&1
ncu -i /tmp/k1b.ncu-rep --page raw --csv > gpurun_out/r3t/k1b_raw.csv 2>&1
cat gpurun_out/r3t/pytest.log
for f in gpurun_out/r3t/c*_st*_*.log gpurun_out/r3t/c2_st*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), round(d['roofline']['gemm_ms_per_forward'],3), round(d['roofline']['kernel_ms_per_forward'],3))" || tail -2 $f; done
