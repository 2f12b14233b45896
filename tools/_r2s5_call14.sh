timeout 1800 python -m pytest tests/test_gpu_pair_lengths.py -x -q > gpurun_out/s5c14_len_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c14_len_tests.log
S="330 420 500 600 700 800 900 1000 1200 1300 1500 1700 1900 2200 2500 2800 3000 3400 3700 4000"
timeout 900 python tools/pad_sweep.py 1 $S > gpurun_out/s5c14_pad_xconv.txt 2>&1
timeout 900 python tools/pad_sweep.py 0 $S > gpurun_out/s5c14_pad_xcorr.txt 2>&1
