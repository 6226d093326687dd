# per-chunk operand arrival / MMA issue time in the c4 recurrence (HS_TRACE_CHUNKS variant build)
mkdir -p gpurun_out/r4d
export HS_LIB_PATH=paper_2307_11339_b200/_lib/libhsrnn_tc.so
timeout 600 python tools/trace_chunks.py c4 > gpurun_out/r4d/chunks2_c4.txt 2>&1
HS_W_TMEM=0 timeout 600 python tools/trace_chunks.py c4 > gpurun_out/r4d/chunks2_c4_wtmem0.txt 2>&1
cat gpurun_out/r4d/chunks2_c4*.txt
