# quick GPU check: tests named by $1 (pytest -k expr or path), plus smoke
set -x
timeout 900 python -m pytest ${1:-tests} -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_quick.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
tail -n 5 gpurun_out/pytest_quick.log gpurun_out/smoke.log
