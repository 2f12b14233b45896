timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_ref.py tests/test_cpp_shim.py -x -q --durations=5 > gpurun_out/c4.log 2>&1
echo rc=$? >> gpurun_out/c4.log
