#!/bin/bash
# Round-2 measurements on one B200: GPU suite, smoke, then each workload as
# its own bench.py run (outputs under gpurun_out/).
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"
run() {  # name timeout args...
  local name=$1 t=$2; shift 2
  timeout $t python "$@" > gpurun_out/r2_$name.json 2> gpurun_out/r2_$name.err; echo "$name rc=$?"
}
[ "$1" == "tests-only" ] && exit 0
run default 900 bench.py --steps 10 --warmup 3
run config0 900 bench.py --workload config0 --steps 10 --warmup 3
run config3 1200 bench.py --workload config3 --steps 5 --warmup 3
run config2 1500 bench.py --workload config2 --steps 3 --warmup 3
