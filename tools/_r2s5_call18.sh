timeout 1800 python -m pytest tests/test_gpu_tiles.py -x -q > gpurun_out/s5c18_tile_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c18_tile_tests.log
timeout 900 python tools/pad_sweep.py 0 4500 6000 8000 > gpurun_out/s5c18_big_xcorr.txt 2>&1
timeout 900 python tools/pad_sweep.py 1 4500 6000 8000 > gpurun_out/s5c18_big_xconv.txt 2>&1
XCB_TILE=0 timeout 900 python tools/pad_sweep.py 0 4500 6000 > gpurun_out/s5c18_big_xcorr_off.txt 2>&1
XCB_TILE=0 timeout 900 python tools/pad_sweep.py 1 4500 6000 > gpurun_out/s5c18_big_xconv_off.txt 2>&1
