#!/bin/bash
# A/B of the cluster NTT at N=2^16 (16-CTA clusters, lib_ab/ntt3_16 built with
# -DHB_NTT3_MAXLOGN=16) against the two-pass kernels: per-mode launch timing,
# the big-ring parity tests, config-3 logits and the config-3 bench.
for v in base ntt3_16; do
  if [ $v == base ]; then export HEAR_B200_LIB=; else export HEAR_B200_LIB=lib_ab/$v/libhear_b200.so; fi
  NTT_MODES_LOGN=16 TAG=$v python tools/ntt_modes.py 8 32
  timeout 900 python -m pytest tests/test_gpu_bigring.py tests/test_gpu_codec.py -q 2>&1 | tail -1
  python tools/diag_big.py c3 2>&1 | tail -4
  timeout 1200 python bench.py --workload config3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab16_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab16_$v.json')); print('$v', round(d['value'],1), d['per_clip_latency']['p50_ms'], d['clocks'])"
done
