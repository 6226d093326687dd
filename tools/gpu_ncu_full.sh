# One ncu --set full capture of the recurrent kernel and of the K1 GEMM (c2 bench workload).
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:recur_tc_kernel -s 2 -c 1 \
  -o gpurun_out/recur_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_recur.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_xproj -s 2 -c 1 \
  -o gpurun_out/gemm_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_gemm.log 2>&1
ls -la gpurun_out
