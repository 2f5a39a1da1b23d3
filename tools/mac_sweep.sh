#!/bin/bash
for shape in "64 16 96 4" "64 8 96 8" "32 48 32 4"; do
  TAG=f64_4x8 python tools/mac_bench.py $shape
  TAG=f64_4x4 HEAR_B200_MAC_TILE=4 python tools/mac_bench.py $shape
  TAG=c3_4x4 HEAR_B200_CHUNK=1 python tools/mac_bench.py $shape
  TAG=c3_2x4 HEAR_B200_CHUNK=1 HEAR_B200_MAC_TILE=2 python tools/mac_bench.py $shape
done
