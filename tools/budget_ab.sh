#!/bin/bash
# Key-switch temporaries budget A/B (GPU box).
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bud_default.json 2> gpurun_out/bud_default.err
for kv in HEAR_B200_KS_BUDGET_GB=12 HEAR_B200_KS_BUDGET_GB=48 HEAR_B200_KS_BUDGET_GB=96; do
  env $kv timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bud_$kv.json 2> gpurun_out/bud_$kv.err
done
true
