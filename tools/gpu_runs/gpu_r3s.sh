set -x
mkdir -p gpurun_out/r3s
for p in 0 20 26 32 38; do if [ $p = 0 ]; then env=""; else env="HS_XP_HEAD=$p"; fi; env $env timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/r3s/c2_p$p.log 2>&1; done
HS_DEBUG_XP=1 timeout 300 python bench.py --no-cpu-baseline --steps 10 2>&1 | grep -i "xp" | tail -4 > gpurun_out/r3s/xpdebug.log
for f in gpurun_out/r3s/c2_*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['roofline']['kernel_ms_per_forward'],4), round(d['roofline']['gemm_ms_per_forward'],4))" || tail -3 $f; done
cat gpurun_out/r3s/xpdebug.log
