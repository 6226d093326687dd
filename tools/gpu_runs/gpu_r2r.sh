# peer pipeline (K4) tests + full suite
set -x
mkdir -p gpurun_out/r2r
export HS_WATCHDOG_MS=20000
timeout 600 python -m pytest tests/test_pipeline_peer.py -m gpu -q -x 2>&1 | tail -30 > gpurun_out/r2r/pytest_peer.log
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/r2r/pytest_gpu.log
cat gpurun_out/r2r/pytest_peer.log gpurun_out/r2r/pytest_gpu.log
