timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_sharded.py tests/test_cpp_shim.py -x -q > gpurun_out/s5c6_multi_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c6_multi_tests.log
