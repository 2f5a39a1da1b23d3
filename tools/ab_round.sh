# GPU tests + bench with the default library, then the same bench with an env override (A/B).
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_a.log 2>&1
[ -n "$AB_ENV" ] && env $AB_ENV timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_b.log 2>&1
timeout 300 python tools/layer_times.py 1d-w64 full 64 > gpurun_out/layers.txt 2>&1
true
