set -x
mkdir -p gpurun_out/r2z
timeout 900 python tools/hybrid_model_check.py c1 gpurun_out/r2z/hybrid_c1.json > gpurun_out/r2z/hybrid_c1.log 2>&1
grep -E '"plan"' gpurun_out/r2z/hybrid_c1.log | cut -c1-250
