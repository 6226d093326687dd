# compute-sanitizer on the production kernel families after the round-2 changes
set -x
mkdir -p gpurun_out/r3d
export HS_WATCHDOG_MS=120000
for tool in racecheck synccheck memcheck; do timeout 1200 compute-sanitizer --tool $tool python tools/sanitize_prod.py > gpurun_out/r3d/$tool.log 2>&1; done
tail -n 4 gpurun_out/r3d/*.log
