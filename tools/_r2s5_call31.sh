timeout 3000 python tools/fuzz_sizes.py 120 7 > gpurun_out/s5c31_fuzz_sizes.log 2>&1; echo rc=$? >> gpurun_out/s5c31_fuzz_sizes.log
