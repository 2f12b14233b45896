python tools/bench_configs.py 2 4 > gpurun_out/c7_cfg24.jsonl 2>&1
XCB_S1_PAIR=1 python tools/bench_configs.py 2 > gpurun_out/c7_cfg2_pair.jsonl 2>&1
XCB_TAIL_SPLIT=0 python tools/bench_configs.py 4 > gpurun_out/c7_cfg4_nosplit.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -x -q -k "scatter or xconv or smooth or config2 or config4 or fuzz or hermitian" > gpurun_out/c7_tests.log 2>&1; echo rc=$? >> gpurun_out/c7_tests.log
XCB_S1_PAIR=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "scatter or xconv or smooth or config2" > gpurun_out/c7_tests_pair.log 2>&1; echo rc=$? >> gpurun_out/c7_tests_pair.log
ncu --set full --clock-control none --import-source on -k regex:"premul" -c 1 -o gpurun_out/c7_s1_cfg4 python tools/profile_case.py smooth 4 > /dev/null 2>&1
XCB_S1_PAIR=1 ncu --set full --clock-control none --import-source on -k regex:"premul" -c 1 -o gpurun_out/c7_s1_cfg2_pair python tools/profile_case.py xconv 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"inv_steer" -c 1 -o gpurun_out/c7_i2_cfg5 python tools/profile_case.py xcorr 5 > /dev/null 2>&1
