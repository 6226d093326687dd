# same-box A/B: commit 06d873a (before the TMEM work) vs HEAD on c4 / c2 / c5
set -x
mkdir -p gpurun_out/r3j
for rep in 1 2; do
  (cd _old && timeout 600 python bench.py --config c4 --no-cpu-baseline --steps 5 > ../gpurun_out/r3j/old_c4_$rep.log 2>&1)
  timeout 600 python bench.py --config c4 --no-cpu-baseline --steps 5 > gpurun_out/r3j/new_c4_$rep.log 2>&1
done
(cd _old && timeout 600 python bench.py --no-cpu-baseline --steps 20 > ../gpurun_out/r3j/old_c2.log 2>&1)
timeout 600 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/r3j/new_c2.log 2>&1
(cd _old && timeout 600 python bench.py --config c5 --no-cpu-baseline --steps 5 > ../gpurun_out/r3j/old_c5.log 2>&1)
timeout 600 python bench.py --config c5 --no-cpu-baseline --steps 5 > gpurun_out/r3j/new_c5.log 2>&1
(cd _old && timeout 600 python bench.py --config c3 --no-cpu-baseline --steps 20 > ../gpurun_out/r3j/old_c3.log 2>&1)
timeout 600 python bench.py --config c3 --no-cpu-baseline --steps 20 > gpurun_out/r3j/new_c3.log 2>&1
for f in gpurun_out/r3j/*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['kernel_ms_per_forward'],3))" || tail -3 $f; done
