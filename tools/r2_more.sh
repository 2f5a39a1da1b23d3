#!/bin/bash
# Full GPU suite after the 2^16 cluster change, config 3 with its CPU
# baseline, and the secondary reference networks.
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pytest_gpu.log
timeout 1500 python bench.py --workload config3 --steps 5 --warmup 3 > gpurun_out/r2_config3.json 2> gpurun_out/r2_config3.err; echo "c3 rc=$?"
timeout 1200 python bench.py --net 2d-w128 --batch 32 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_2dw128.json 2> gpurun_out/r2_2dw128.err; echo "2d rc=$?"
timeout 1200 python bench.py --mode hear --batch 64 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_hear.json 2> gpurun_out/r2_hear.err; echo "hear rc=$?"
