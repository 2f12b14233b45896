timeout 900 python -m pytest tests/test_gpu_cpair.py -x -q > gpurun_out/s5c2_cpair_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c2_cpair_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_detect.py tests/test_contour.py -x -q -k "scatter or config2 or full_size_sampled or detect or contour or smooth or config4" > gpurun_out/s5c2_scatter_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c2_scatter_tests.log
timeout 400 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/s5c2_bench_cfg2.json 2> gpurun_out/s5c2_bench_cfg2.err
XCB_CPAIR=0 timeout 400 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/s5c2_bench_cfg2_nocpair.json 2> gpurun_out/s5c2_bench_cfg2_nocpair.err
