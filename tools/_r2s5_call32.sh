timeout 1800 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_cpair.py -x -q > gpurun_out/s5c32_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c32_tests.log
