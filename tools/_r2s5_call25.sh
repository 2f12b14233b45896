timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s5c25_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c25_gpu_tests.log
for c in 1 2; do timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu > gpurun_out/s5c25_bench_cfg$c.json 2> gpurun_out/s5c25_bench_cfg$c.err; done
for c in 1 2; do XCB_PREP=1 timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu > gpurun_out/s5c25_bench_cfg${c}_prep.json 2> gpurun_out/s5c25_bench_cfg${c}_prep.err; done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/s5c25_bench_cfg5.json 2> gpurun_out/s5c25_bench_cfg5.err
XCB_PREP=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/s5c25_bench_cfg5_prep.json 2> gpurun_out/s5c25_bench_cfg5_prep.err
