# final HEAD evidence after the hidden-layer fp16 K1: GPU suite, smoke, bench c2 (default) + c3/c4/c5, reference arm, c2 launch list
mkdir -p gpurun_out/r5p
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/r5p/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5p/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r5p/bench_c2.log 2>&1
for c in c3 c4 c5; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 > gpurun_out/r5p/bench_$c.log 2>&1; done
timeout 600 python bench.py --config c5 --global-batch 32 --no-cpu-baseline --steps 5 > gpurun_out/r5p/bench_c5_shard32.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r5p/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r5p/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r5p/b_ncu_c2.log 2>&1
for f in gpurun_out/r5p/bench_c*.log; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['roofline']['kernel_ms_per_forward'],3), round(d['e2e']['value'],1) if d.get('e2e') else None, d['clocks'])"; done
cat gpurun_out/r5p/pytest_gpu.log gpurun_out/r5p/smoke.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_xproj -s 2 -c 3 -o /tmp/ncu_k1 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r5p/ncu_k1.log 2>&1
ncu -i /tmp/ncu_k1.ncu-rep --page raw --csv > gpurun_out/r5p/ncu_k1_raw.csv 2>&1
