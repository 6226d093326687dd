# Round GPU evidence: pytest -m gpu, smoke, bench (ours + reference arm), ncu
# launch list + full captures of the recurrent kernel and K1, compute-sanitizer.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
for c in c3 c4 c5; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 > gpurun_out/b_$c.log 2>&1; done
timeout 300 python tools/c1_latency.py > gpurun_out/c1_latency.json 2>/dev/null
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:recur_tc -s 2 -c 1 -o gpurun_out/recur_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_recur.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_xproj -s 2 -c 1 -o gpurun_out/gemm_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_gemm.log 2>&1
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_case.py > gpurun_out/racecheck.log 2>&1
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_case.py > gpurun_out/synccheck.log 2>&1
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_case.py > gpurun_out/memcheck.log 2>&1
tail -n 3 gpurun_out/*.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_torchrun.log 2>&1
tail -n 2 gpurun_out/b_torchrun.log
