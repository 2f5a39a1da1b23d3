#!/bin/bash
# Clips-per-step sweep of the bench default and the secondary workloads (GPU box).
for b in 96 160 192 256; do
  timeout 600 python bench.py --batch $b --no-cpu-baseline > gpurun_out/sw_b$b.json 2> gpurun_out/sw_b$b.err
done
timeout 600 python bench.py --net 2d-w128 --batch 32 --no-cpu-baseline > gpurun_out/res_2dw128.json 2> gpurun_out/res_2dw128.err
timeout 600 python bench.py --net 2d-w128 --batch 64 --no-cpu-baseline > gpurun_out/res_2dw128_b64.json 2> gpurun_out/res_2dw128_b64.err
timeout 600 python bench.py --mode hear --batch 32 --no-cpu-baseline > gpurun_out/res_hear.json 2> gpurun_out/res_hear.err
timeout 600 python bench.py --mode hear --batch 64 --no-cpu-baseline > gpurun_out/res_hear_b64.json 2> gpurun_out/res_hear_b64.err
true
