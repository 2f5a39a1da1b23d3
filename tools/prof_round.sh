#!/bin/bash
# Round profiling pass (GPU box): launch list of one eager 1d-w64 step and
# ncu --set full captures of the top kernels.  Summaries: tools/ncu_summary.py
set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
python tools/step_profile.py 1d-w64 full 64 > gpurun_out/p2_sp.log 2>&1 || exit 1
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/p2_launches_b64.csv python tools/step_profile.py 1d-w64 full 64 > gpurun_out/p2_ncu_list.log 2>&1
python tools/roofline_probe.py > gpurun_out/p2_roof.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_ntt3 -s 3 -c 1 -o gpurun_out/p2_full_roofline python tools/roofline_probe.py > gpurun_out/p2_ncu_roof.log 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_ntt3_fwd<hb::PolF64, .int.14, .int.1>" -s 4 -c 1 -o gpurun_out/p2_full_lift python tools/step_profile.py 1d-w64 full 64 > gpurun_out/p2_ncu_lift.log 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_ntt3_inv -s 8 -c 1 -o gpurun_out/p2_full_inv python tools/step_profile.py 1d-w64 full 64 > gpurun_out/p2_ncu_inv.log 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_mac_pipe<.int.8, .int.4, .int.2, .int.4, .int.3" -s 6 -c 1 -o gpurun_out/p2_full_ksgemm python tools/step_profile.py 1d-w64 full 64 > gpurun_out/p2_ncu_ksg.log 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_mac_pipe<.int.8, .int.4, .int.1, .int.8, .int.3" -s 0 -c 1 -o gpurun_out/p2_full_mac python tools/step_profile.py 1d-w64 full 64 > gpurun_out/p2_ncu_mac.log 2>&1
ls gpurun_out
