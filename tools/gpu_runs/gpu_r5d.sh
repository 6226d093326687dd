# r5c after: hybrid dispatch setup before the clock (events, device/stream context), run_cells(stream=)
mkdir -p gpurun_out/r5d
timeout 600 python -m pytest tests/test_gpu_cells.py tests/test_executor.py tests/test_gpu_integration.py -q -x 2>&1 | tail -3 > gpurun_out/r5d/pytest.log
timeout 300 python tools/probe/hybrid_spans.py c1 > gpurun_out/r5d/hspans.txt 2>&1
timeout 300 python tools/probe/hybrid_spans.py c1 first >> gpurun_out/r5d/hspans.txt 2>&1
timeout 600 python tools/hybrid_model_check.py c1 gpurun_out/r5d/hybrid_c1.json > gpurun_out/r5d/hybrid_c1.log 2>&1
timeout 900 python tools/hybrid_model_check.py c3 gpurun_out/r5d/hybrid_c3.json --seq 64 > gpurun_out/r5d/hybrid_c3.log 2>&1
cat gpurun_out/r5d/pytest.log; grep -h '"plan"' gpurun_out/r5d/hybrid_c*.log | grep -v '^ ' | cut -c1-300; head -30 gpurun_out/r5d/hspans.txt
