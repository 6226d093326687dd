# hybrid model check (c1, c3 T=64); c2 single-layer W-streaming step time at S=2 (wave feasibility probe)
set -x
mkdir -p gpurun_out/r2o
timeout 900 python tools/hybrid_model_check.py c1 gpurun_out/r2o/hybrid_c1.json > gpurun_out/r2o/hybrid_c1.log 2>&1
timeout 1500 python tools/hybrid_model_check.py c3 gpurun_out/r2o/hybrid_c3.json --seq 64 > gpurun_out/r2o/hybrid_c3.log 2>&1
for cfg in "HS_FORCE_STREAM=1 HS_FORCE_S=2 HS_TWO_GROUPS=0 HS_XP_STREAM=0" "HS_FORCE_STREAM=1 HS_TWO_GROUPS=0 HS_XP_STREAM=0" "HS_TWO_GROUPS=0 HS_XP_STREAM=0" "HS_XP_STREAM=0"; do
  env $cfg timeout 300 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > /tmp/b.log 2>&1
  echo "$cfg" >> gpurun_out/r2o/stream_probe.log
  python -c "import json; d=json.loads(open('/tmp/b.log').read().strip().splitlines()[-1]); print(d['plan'], d['roofline']['kernel_ms_per_forward'], d['value'])" >> gpurun_out/r2o/stream_probe.log 2>&1 || tail -3 /tmp/b.log >> gpurun_out/r2o/stream_probe.log
done
cat gpurun_out/r2o/stream_probe.log
tail -n 12 gpurun_out/r2o/hybrid_c1.log gpurun_out/r2o/hybrid_c3.log
