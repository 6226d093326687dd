# A/B helper: pytest -m gpu, then bench configs with env $ABVAR=1/0 (device + e2e values), timeline
set -x
V=${ABVAR:-HS_K1_CHUNKED}
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/ab_pytest.log
for c in ${ABCFG:-c2 c3}; do for v in ${ABVALS:-1 0 1 0}; do env $V=$v timeout 300 python bench.py --config $c --no-cpu-baseline --steps 30 > gpurun_out/ab_${c}_$v.log 2>&1; echo "$c $V=$v $(grep -o "\"value\": [0-9.]*" gpurun_out/ab_${c}_$v.log | head -2 | tr "\n" " ")"; done; done
timeout 300 python tools/timeline.py c2 > gpurun_out/timeline_c2.txt 2>&1
cat gpurun_out/ab_pytest.log
