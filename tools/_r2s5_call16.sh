timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s5c16_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c16_gpu_tests.log
S="100 200 330 500 700 900 1000 1200 1500 1700 1900 2200 2500 2800 3000 3400 3700 4000 4200"
timeout 900 python tools/pad_sweep.py 1 $S > gpurun_out/s5c16_pad_xconv.txt 2>&1
timeout 900 python tools/pad_sweep.py 0 $S > gpurun_out/s5c16_pad_xcorr.txt 2>&1
XCB_PAD_RULE=0 timeout 900 python tools/pad_sweep.py 1 $S > gpurun_out/s5c16_pad_xconv_old.txt 2>&1
XCB_PAD_RULE=0 timeout 900 python tools/pad_sweep.py 0 $S > gpurun_out/s5c16_pad_xcorr_old.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/s5c16_bench_cfg5.json 2> gpurun_out/s5c16_bench_cfg5.err
for c in 1 2 3 4; do timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu > gpurun_out/s5c16_bench_cfg$c.json 2> gpurun_out/s5c16_bench_cfg$c.err; done
