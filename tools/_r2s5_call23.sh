timeout 400 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu > gpurun_out/s5c23_bench_cfg1.json 2> gpurun_out/s5c23_bench_cfg1.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_ref.py -x -q > gpurun_out/s5c23_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c23_tests.log
timeout 600 python tools/pad_sweep.py 0 100 150 200 256 > gpurun_out/s5c23_small_xcorr.txt 2>&1
timeout 600 python tools/pad_sweep.py 1 100 150 200 256 > gpurun_out/s5c23_small_xconv.txt 2>&1
