HEAR_B200_PREPERM=1 timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
TAG=base python tools/ks_probe.py > gpurun_out/ks.log 2>&1
TAG=pp_gemm HEAR_B200_PREPERM=1 python tools/ks_probe.py >> gpurun_out/ks.log 2>&1
TAG=pp_inner2 HEAR_B200_PREPERM=1 HEAR_B200_KS_GEMM_MIN=1000 python tools/ks_probe.py >> gpurun_out/ks.log 2>&1
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_a.log 2>&1
HEAR_B200_PREPERM=1 timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_b.log 2>&1
