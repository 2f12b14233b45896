timeout 1800 python -m pytest tests/test_gpu_guards.py -x -q > gpurun_out/s5c22_guards.log 2>&1; echo rc=$? >> gpurun_out/s5c22_guards.log
