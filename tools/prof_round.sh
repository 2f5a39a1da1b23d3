set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
timeout 300 python tools/layer_times.py 1d-w64 full 64 > gpurun_out/layers.txt 2>&1
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/launches_b64.csv python tools/step_profile.py 1d-w64 full 64 > gpurun_out/ncu_list.log 2>&1
for k in k_ntt2_blocks k_ntt2_cols k_ks_inner2 k_mac_gemm; do
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$k --launch-skip 40 -c 1 -o gpurun_out/full_$k python tools/step_profile.py 1d-w64 full 64 > gpurun_out/ncu_full_$k.log 2>&1
done
ls -la gpurun_out
