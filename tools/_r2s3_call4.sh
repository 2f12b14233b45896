timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3c4_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s3c4_gpu_tests.log
timeout 600 python tools/ab_kernels.py --case "xcorr 5 1" --regex "ilv" sc mix > gpurun_out/s3c4_ab_cfg5.txt 2>&1
timeout 600 python tools/ab_kernels.py --case "anglemax 3 1" --regex "ilv|angle" sc mix > gpurun_out/s3c4_ab_cfg3.txt 2>&1
timeout 600 python tools/ab_kernels.py --case "xcorr 1 1" --regex "." sc mix > gpurun_out/s3c4_ab_cfg1.txt 2>&1
for c in 5 2 4 3 1; do timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/s3c4_bench_cfg$c.json 2> gpurun_out/s3c4_bench_cfg$c.err; done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "rotation_matches_oracle_fast_path or smooth_matches_oracle or config1_full_size or config2_reduced" > gpurun_out/s3c4_memcheck.log 2>&1; echo rc=$? >> gpurun_out/s3c4_memcheck.log
