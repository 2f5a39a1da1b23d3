#!/bin/bash
# NTT kernel A/B on the GPU box: per-mode launch timing, determinism digests
# under load, and the bench line, for the in-tree build and lib_ab/<tag>.
tag=$1
for v in base $tag; do
  if [ $v == base ]; then export HEAR_B200_LIB=; else export HEAR_B200_LIB=lib_ab/$v/libhear_b200.so; fi
  for i in 1 2; do TAG=$v python tools/ntt_modes.py 12 64; done
  python tools/ntt3_check.py > gpurun_out/ab_digest_$v.txt 2>&1
  timeout 900 python -m pytest tests/test_gpu_ntt_load.py -q 2>&1 | tail -1
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_bench_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_bench_$v.json')); print('$v', round(d['value'],1), d['clocks'])"
done
diff gpurun_out/ab_digest_base.txt gpurun_out/ab_digest_$tag.txt > /dev/null && echo "digests identical" || echo "DIGESTS DIFFER"
