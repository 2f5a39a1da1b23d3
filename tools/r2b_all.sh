#!/bin/bash
# Round-2 final measurements on one B200: every workload as its own bench.py
# run (outputs gpurun_out/r2b_*.json), B=1 latency knobs, stream and primitives.
mkdir -p gpurun_out
run() {  # name timeout args...
  local name=$1 t=$2; shift 2
  timeout $t python "$@" > gpurun_out/r2b_$name.json 2> gpurun_out/r2b_$name.err; echo "$name rc=$?"
}
run config0 900 bench.py --workload config0 --steps 10 --warmup 3
run config3 1500 bench.py --workload config3 --steps 5 --warmup 3
run config2 1500 bench.py --workload config2 --steps 3 --warmup 3
run 2dw128 1200 bench.py --net 2d-w128 --batch 32 --steps 5 --warmup 3 --no-cpu-baseline
run hear 1200 bench.py --mode hear --batch 64 --steps 5 --warmup 3 --no-cpu-baseline
HEAR_B200_LAZY_MIN=8 run b1eager 900 bench.py --steps 3 --warmup 3 --no-cpu-baseline
HEAR_B200_LAZY_MIN=1 HEAR_B200_KS_FUSED_MIN=40 run b1lazyfused 900 bench.py --steps 3 --warmup 3 --no-cpu-baseline
HEAR_B200_KS_FUSED_MIN=40 run b1fused 900 bench.py --steps 3 --warmup 3 --no-cpu-baseline
timeout 900 python tools/stream_bench.py > gpurun_out/r2b_stream_config4.json 2> gpurun_out/r2b_stream.err; echo "stream rc=$?"
python tools/bench_summary.py gpurun_out/r2b_config0.json gpurun_out/r2b_config3.json gpurun_out/r2b_config2.json gpurun_out/r2b_2dw128.json gpurun_out/r2b_hear.json gpurun_out/r2b_b1eager.json gpurun_out/r2b_b1lazyfused.json gpurun_out/r2b_b1fused.json
