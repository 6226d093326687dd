set -x
mkdir -p gpurun_out/r2s
export HS_WATCHDOG_MS=20000
timeout 900 python -m pytest tests/test_pipeline_peer.py -m gpu -q 2>&1 | tail -30 > gpurun_out/r2s/pytest_peer.log
cat gpurun_out/r2s/pytest_peer.log
