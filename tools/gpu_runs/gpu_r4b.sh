# c4 per-phase trace, W ring 4 vs 5
mkdir -p gpurun_out/r4b
for r in 4 5; do
  HS_W_RING=$r TRACE_S=2 timeout 600 python tools/trace_recur.py c4 /tmp/tr_c4_$r.bin > gpurun_out/r4b/trace_c4_ring$r.txt 2>&1
done
cat gpurun_out/r4b/trace_c4_ring*.txt
