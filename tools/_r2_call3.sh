set -x
timeout 600 python -m pytest tests/test_gpu_decompose.py tests/test_detect.py tests/test_contour.py tests/test_lic.py -x -q > gpurun_out/r2c3_decomp.log 2>&1; echo rc=$? >> gpurun_out/r2c3_decomp.log
timeout 600 python tools/ab_kernels.py --case "xconv 2" --regex "premul|mac|inv_out" cur p8_12_12 p8_16_9 > gpurun_out/r2c3_ab_cfg2.txt 2>&1
for v in p8_12_12 p8_16_9; do XCB_LIB_OVERRIDE=paper_2006_13188_b200/lib/ab/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "scatter or xconv or config2 or smooth" > gpurun_out/r2c3_par_$v.log 2>&1; echo rc=$? >> gpurun_out/r2c3_par_$v.log; done
timeout 600 python tools/ab_kernels.py --case "xcorr 5" --regex "inv_steer" cur > gpurun_out/r2c3_ab_cfg5_i2.txt 2>&1
