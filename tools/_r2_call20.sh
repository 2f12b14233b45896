timeout 600 python tools/ab_kernels.py --case "xconv 2" --regex "premul|mac|inv_out" head s1occ > gpurun_out/r2c20_ab_cfg2.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py -x -q -k "scatter or xconv or config2 or fuzz" > gpurun_out/r2c20_par.log 2>&1; echo rc=$? >> gpurun_out/r2c20_par.log
