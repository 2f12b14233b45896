timeout 600 python tools/pad_sweep.py 1 900 1000 1100 1900 2000 2100 3400 3900 4000 4200 > gpurun_out/s5c9_pad_xconv.txt 2>&1
timeout 600 python tools/pad_sweep.py 0 900 1000 1100 1900 2000 2100 3400 3900 4000 4200 > gpurun_out/s5c9_pad_xcorr.txt 2>&1
