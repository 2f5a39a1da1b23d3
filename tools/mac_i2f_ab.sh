#!/bin/bash
# A/B of the GEMM operand conversion (lib_ab built with -DHB_MAC_I2F).
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/i2f_a1.json 2> gpurun_out/i2f_a1.err
HEAR_B200_LIB=$PWD/lib_ab/libhear_b200.so timeout 600 python bench.py --no-cpu-baseline > gpurun_out/i2f_b1.json 2> gpurun_out/i2f_b1.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/i2f_a2.json 2> gpurun_out/i2f_a2.err
HEAR_B200_LIB=$PWD/lib_ab/libhear_b200.so timeout 600 python bench.py --no-cpu-baseline > gpurun_out/i2f_b2.json 2> gpurun_out/i2f_b2.err
HEAR_B200_LIB=$PWD/lib_ab/libhear_b200.so timeout 900 python -m pytest tests/test_gpu_ckks.py tests/test_gpu_pipeline.py -m gpu -x -q > gpurun_out/i2f_tests.log 2>&1; echo rc=$? >> gpurun_out/i2f_tests.log
true
