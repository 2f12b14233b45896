XCB_TC_VARIANT=3 XCB_TC_TRACE=1 timeout 120 python tools/profile_case.py anglemax 3 > gpurun_out/r2c16_trace.txt 2>&1
