# Round-2 re-entry check: full -m gpu suite, smoke, benches c2..c5 and the reference arm.
set -x
mkdir -p gpurun_out/r2k
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r2k/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2k/bench_c2.log 2>&1
for c in c3 c4 c5; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 > gpurun_out/r2k/bench_$c.log 2>&1; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2k/bench_ref.log 2>&1
tail -n 3 gpurun_out/r2k/*.log
