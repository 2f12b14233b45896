S="330 420 500 600 700 800 1200 1300 1500 1700 2200 2500 3000 3400"
timeout 900 python tools/pad_sweep.py 1 $S > gpurun_out/s5c13_pad_xconv.txt 2>&1
timeout 900 python tools/pad_sweep.py 0 $S > gpurun_out/s5c13_pad_xcorr.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s5c13_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c13_gpu_tests.log
