timeout 600 python tools/pad_sweep.py 1 800 900 1000 1700 1900 2000 3400 3900 4000 > gpurun_out/s5c10_pad_xconv.txt 2>&1
timeout 600 python tools/pad_sweep.py 0 800 900 1000 1700 1900 2000 3400 3900 4000 > gpurun_out/s5c10_pad_xcorr.txt 2>&1
XCB_PAD_PAIR=0 timeout 600 python tools/pad_sweep.py 1 800 1700 > gpurun_out/s5c10_pad_xconv_off.txt 2>&1
XCB_PAD_PAIR=0 timeout 600 python tools/pad_sweep.py 0 800 1700 > gpurun_out/s5c10_pad_xcorr_off.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s5c10_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c10_gpu_tests.log
