for v in base ntt3_15; do
  if [ $v == base ]; then export HEAR_B200_LIB=; else export HEAR_B200_LIB=lib_ab/$v/libhear_b200.so; fi
  NTT_MODES_LOGN=15 TAG=$v python tools/ntt_modes.py 12 64
  timeout 900 python -m pytest tests/test_gpu_bigring.py -q 2>&1 | tail -1
  python tools/diag_big.py c2 2>&1 | tail -4
  timeout 1200 python bench.py --workload config2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab15_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab15_$v.json')); print('$v', round(d['value'],1), d['per_clip_latency']['p50_ms'], d['clocks'])"
done
