#!/bin/bash
# Round results pass (GPU box): the bench default, its reference arm, the
# secondary workloads.  Output lines land in gpurun_out/res_*.json
timeout 600 python bench.py > gpurun_out/res_default.json 2> gpurun_out/res_default.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/res_ref.json 2> gpurun_out/res_ref.err
timeout 600 python bench.py --net 2d-w128 --batch 32 --no-cpu-baseline > gpurun_out/res_2dw128.json 2> gpurun_out/res_2dw128.err
timeout 600 python bench.py --mode hear --batch 32 --no-cpu-baseline > gpurun_out/res_hear.json 2> gpurun_out/res_hear.err
timeout 600 python bench.py --batch 128 --no-cpu-baseline > gpurun_out/res_b128.json 2> gpurun_out/res_b128.err
timeout 900 python tools/primitives_bench.py > gpurun_out/res_primitives.json 2> gpurun_out/res_primitives.err
timeout 900 python tools/stream_bench.py > gpurun_out/res_stream.json 2> gpurun_out/res_stream.err
true
