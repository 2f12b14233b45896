XCB_FUZZ_CASES=1000 timeout 3000 python -m pytest tests/test_gpu_fuzz.py -x -q > gpurun_out/s5c30_fuzz1000.log 2>&1; echo rc=$? >> gpurun_out/s5c30_fuzz1000.log
