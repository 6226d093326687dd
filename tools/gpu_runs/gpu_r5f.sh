# ncu --set full at HEAD: c2 recurrence (recur_tc2), c2 K1 head (gemm_xproj_persistent / dyn), c4 recurrence; raw CSV exported on the box
mkdir -p gpurun_out/r5f
cap() {  # name, kernel regex, skip, bench args...
  local n=$1 k=$2 sk=$3; shift 3
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s $sk -c 1 -o /tmp/ncu_$n -f python bench.py "$@" --no-cpu-baseline > gpurun_out/r5f/ncu_$n.log 2>&1
  ncu -i /tmp/ncu_$n.ncu-rep --page raw --csv > gpurun_out/r5f/ncu_${n}_raw.csv 2>&1
  ncu -i /tmp/ncu_$n.ncu-rep --page details --csv > gpurun_out/r5f/ncu_${n}_details.csv 2>&1
}
cap c2_recur recur_tc2 2 --steps 1 --warmup 3
cap c2_k1 gemm_xproj_persistent 2 --steps 1 --warmup 3
cap c2_k1dyn gemm_xproj_dyn 4 --steps 1 --warmup 3
cap c4_recur recur_tc_kernel 8 --config c4 --steps 1 --warmup 3
ls -la gpurun_out/r5f
