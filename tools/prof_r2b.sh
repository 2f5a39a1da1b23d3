#!/bin/bash
# Round-2 (second half) profiling pass on the GPU box: launch list of one
# eager 1d-w64 step at the bench's 128 clips, and ncu --set full captures of
# the top kernels.  Summaries: tools/launch_summary2.py, tools/ncu_summary.py
set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
B=${1:-128}
python tools/step_profile.py 1d-w64 full $B > gpurun_out/p3_sp.log 2>&1 || exit 1
timeout 1500 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/p3_launches_b$B.csv python tools/step_profile.py 1d-w64 full $B > gpurun_out/p3_ncu_list.log 2>&1
python tools/roofline_probe.py > gpurun_out/p3_roof.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_ks3 -s 3 -c 1 -o gpurun_out/p3_full_ks3 python tools/roofline_probe.py > gpurun_out/p3_ncu_roof.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_mac_pipe<.int.8, .int.4, .int.1, .int.4, .int.3, .int.1" -s 2 -c 1 -o gpurun_out/p3_full_ksgemm python tools/step_profile.py 1d-w64 full $B > gpurun_out/p3_ncu_ksg.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_mac_pipe<.int.4, .int.4, .int.2, .int.2, .int.4, .int.0, .int.0, .int.1" -s 0 -c 1 -o gpurun_out/p3_full_mac python tools/step_profile.py 1d-w64 full $B > gpurun_out/p3_ncu_mac.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_ntt3_inv -s 8 -c 1 -o gpurun_out/p3_full_inv python tools/step_profile.py 1d-w64 full $B > gpurun_out/p3_ncu_inv.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_ntt3_fwd<hb::PolF64, .int.14, .int.5>" -s 1 -c 1 -o gpurun_out/p3_full_mdr python tools/step_profile.py 1d-w64 full $B > gpurun_out/p3_ncu_mdr.log 2>&1
ls -la gpurun_out | tail -20
