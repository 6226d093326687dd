# c4 pipeline mode N=1 (peer vs nccl hand-off), c5 strong-scaling shard at N=1 with global batch 32 (8-way c5 shard size)
set -x
mkdir -p gpurun_out/r2t
timeout 600 python bench.py --config c4 --mode pipeline --handoff peer --steps 3 --warmup 3 > gpurun_out/r2t/c4_pipe_peer.log 2>&1
timeout 600 python bench.py --config c4 --mode pipeline --handoff nccl --steps 3 --warmup 3 > gpurun_out/r2t/c4_pipe_nccl.log 2>&1
timeout 600 python bench.py --config c5 --global-batch 32 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r2t/c5_gb32.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --config c4 --mode pipeline --gpus 1 --steps 3 --warmup 3 > gpurun_out/r2t/c4_pipe_torchrun.log 2>&1
tail -n 2 gpurun_out/r2t/*.log | cut -c1-600
