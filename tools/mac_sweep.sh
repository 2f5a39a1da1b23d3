#!/bin/bash
# MAC kernel variants on the conv shapes of 1d-w64 (dev tool)
for shape in "64 16 96 4" "64 8 96 8" "64 32 8 10" "64 4 64 6"; do
  TAG=pipe_f64 python tools/mac_bench.py $shape
  TAG=reg_f64 HEAR_B200_MAC_PIPE=0 python tools/mac_bench.py $shape
done
