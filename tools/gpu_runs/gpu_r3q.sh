set -x
mkdir -p gpurun_out/r3q
export HS_WATCHDOG_MS=20000
timeout 900 python -m pytest tests/test_pipeline_peer.py -m gpu -q 2>&1 | tail -5 > gpurun_out/r3q/peer.log
cat gpurun_out/r3q/peer.log
