S="100 150 200 330 420 600 700 800 1200 1300 1500 1700 2200 2500 3000"
timeout 900 python tools/pad_sweep.py 1 $S > gpurun_out/s5c11_pad_xconv_new.txt 2>&1
XCB_PAD_RULE=0 timeout 900 python tools/pad_sweep.py 1 $S > gpurun_out/s5c11_pad_xconv_old.txt 2>&1
timeout 900 python tools/pad_sweep.py 0 $S > gpurun_out/s5c11_pad_xcorr_new.txt 2>&1
XCB_PAD_RULE=0 timeout 900 python tools/pad_sweep.py 0 $S > gpurun_out/s5c11_pad_xcorr_old.txt 2>&1
