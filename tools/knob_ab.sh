#!/bin/bash
# Re-measure the opt-in knobs at HEAD against the default (GPU box).
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_default.json 2> gpurun_out/ab_default.err
for kv in HEAR_B200_BATCH_HOIST=1 HEAR_B200_KS_FUSED=1 HEAR_B200_FOLD_C0=1 HEAR_B200_PDL=1 HEAR_B200_GEMM_TILE=48; do
  env $kv timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_$kv.json 2> gpurun_out/ab_$kv.err
done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_default2.json 2> gpurun_out/ab_default2.err
true
