set -x
HS_WAVE_2SM=0 python tools/_wave_l2.py 2>&1 | head -20 > gpurun_out/trace_l2.txt
HS_WAVE=0 HS_FORCE_S=2 TRACE_S=2 HS_RECUR_TRACE=gpurun_out/t.bin python tools/trace_recur.py c3 > gpurun_out/trace_c3_s2.txt 2>&1
HS_WAVE=0 TRACE_S=4 HS_RECUR_TRACE=gpurun_out/t.bin python tools/trace_recur.py c3 > gpurun_out/trace_c3_s4.txt 2>&1
cat gpurun_out/trace_l2.txt gpurun_out/trace_c3_s2.txt gpurun_out/trace_c3_s4.txt
