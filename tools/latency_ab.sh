#!/bin/bash
# B=1 latency knobs at HEAD (GPU box): key-switch GEMM threshold and PDL.
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/lat_default.json 2> gpurun_out/lat_default.err
for kv in HEAR_B200_KS_GEMM_MIN=1 HEAR_B200_KS_GEMM_MIN=2 HEAR_B200_KS_GEMM_MIN=4 HEAR_B200_KS_GEMM_MIN=16 HEAR_B200_PDL=1; do
  env $kv timeout 600 python bench.py --no-cpu-baseline > gpurun_out/lat_$kv.json 2> gpurun_out/lat_$kv.err
done
true
