timeout 900 python -m pytest tests/test_gpu_tcn.py -q 2>&1 | tail -2
timeout 900 python bench.py --workload config0 --steps 10 --warmup 3 > gpurun_out/r2_config0.json 2> gpurun_out/r2_config0.err; echo c0 $?
timeout 1200 python bench.py --workload config3 --steps 5 --warmup 3 > gpurun_out/r2_config3.json 2> gpurun_out/r2_config3.err; echo c3 $?
timeout 900 python tools/stream_bench.py > gpurun_out/r2_stream_config4.json 2> gpurun_out/r2_stream.err; echo st $?
bash tools/prof_aux.sh
