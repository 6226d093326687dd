# Code-path check of the multi-rank bench modes on a one-GPU box: every rank on cuda:0, gloo for the
# collectives (the --handoff nccl pipeline needs NCCL: gloo cannot send CUDA tensors, so it fails here).
# Not a measurement (ranks time-slice one GPU).
set -x
mkdir -p gpurun_out/mr
export HS_BENCH_ONE_DEVICE=1 HS_BENCH_BACKEND=gloo
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 2 "${@:2}"; }
run 29601 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/mr/shard.log 2>&1
run 29602 --config c5 --global-batch 64 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/mr/strong.log 2>&1
run 29603 --config c4 --mode pipeline --steps 2 --warmup 3 > gpurun_out/mr/pipe_peer.log 2>&1
run 29604 --config c4 --mode pipeline --handoff nccl --steps 2 --warmup 3 > gpurun_out/mr/pipe_chunks.log 2>&1
run 29605 --impl reference --steps 2 --warmup 3 > gpurun_out/mr/ref.log 2>&1
for f in gpurun_out/mr/*.log; do echo "== $f"; tail -n 2 $f | cut -c1-400; done
