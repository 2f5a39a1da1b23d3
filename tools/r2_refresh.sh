#!/bin/bash
# Refresh after kernel changes: GPU suite, smoke, default bench, config 2.
bash tools/final_round.sh
timeout 1500 python bench.py --workload config2 --steps 3 --warmup 3 > gpurun_out/r2_config2.json 2> gpurun_out/r2_config2.err; echo "c2 rc=$?"
