timeout 1800 python -m pytest tests/test_gpu_cpair.py tests/test_gpu_pair_lengths.py -x -q > gpurun_out/s5c15_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c15_tests.log
timeout 900 python tools/pad_sweep.py 1 3400 3700 4000 4200 > gpurun_out/s5c15_pad_xconv.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s5c15_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c15_gpu_tests.log
