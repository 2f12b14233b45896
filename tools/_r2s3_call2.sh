timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fft.py tests/test_gpu_ref.py tests/test_gpu_smooth_pack.py tests/test_gpu_anglemax_tc.py -x -q > gpurun_out/s3c2_par.log 2>&1; echo rc=$? >> gpurun_out/s3c2_par.log
timeout 600 python tools/ab_kernels.py --case "xcorr 5 1" --regex "ilv|fwd|F1|F2" sc f2 > gpurun_out/s3c2_ab_cfg5.txt 2>&1
timeout 600 python tools/ab_kernels.py --case "xconv 2 1" --regex "ilv|fast" sc f2 > gpurun_out/s3c2_ab_cfg2.txt 2>&1
timeout 600 python tools/ab_kernels.py --case "smooth 4 1" --regex "ilv|fast" sc f2 > gpurun_out/s3c2_ab_cfg4.txt 2>&1
timeout 600 python tools/ab_kernels.py --case "anglemax 3 1" --regex "ilv|angle" sc f2 > gpurun_out/s3c2_ab_cfg3.txt 2>&1
for c in 5 2 4 3 1; do timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/s3c2_bench_cfg$c.json 2> gpurun_out/s3c2_bench_cfg$c.err; done
