timeout 1800 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_anglemax_tc.py tests/test_gpu_fullsize.py -x -q > gpurun_out/s5c21_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c21_tests.log
timeout 400 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu > gpurun_out/s5c21_bench_cfg3.json 2> gpurun_out/s5c21_bench_cfg3.err
