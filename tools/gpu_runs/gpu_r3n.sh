set -x
mkdir -p gpurun_out/r3n
for rep in 1 2; do for n in 4 8 16 32; do HS_DRAIN_CHUNKS=$n timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/r3n/c2_n${n}_$rep.log 2>&1; done; done
for f in gpurun_out/r3n/c*.log; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), round(d['e2e']['single_request_p50_ms'],3))" || tail -3 $f; done
