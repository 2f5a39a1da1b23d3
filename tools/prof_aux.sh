#!/bin/bash
# ncu captures of the codec FFT, base conversion and integer-policy kernels (GPU box).
python tools/prof_aux.py > gpurun_out/p3_aux.log 2>&1 || exit 1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/p3_launches_aux.csv python tools/prof_aux.py > gpurun_out/p3_list.log 2>&1
for k in k_fft_cols k_fft_rows k_bconv k_ks_inner2 k_ntt2_cols k_ntt2_blocks; do
  timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/p3_full_$k python tools/prof_aux.py > gpurun_out/p3_ncu_$k.log 2>&1
done
ls gpurun_out | grep p3_
