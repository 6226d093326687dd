# HEAD check after the hybrid-executor cleanup: GPU suite, smoke, c2 bench, hybrid model check c1
mkdir -p gpurun_out/r5j
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/r5j/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5j/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r5j/bench_c2.log 2>&1
timeout 600 python tools/hybrid_model_check.py c1 gpurun_out/r5j/hybrid_c1.json > gpurun_out/r5j/hybrid_c1.log 2>&1
cat gpurun_out/r5j/pytest_gpu.log gpurun_out/r5j/smoke.log
python -c "import json; d=json.loads(open('gpurun_out/r5j/bench_c2.log').read().strip().splitlines()[-1]); print('c2', round(d['value'],1), round(d['e2e']['value'],1), d['clocks'], d['cpu_baseline']['value'])"
grep '"plan"' gpurun_out/r5j/hybrid_c1.log | grep -v '^ ' | cut -c1-220
