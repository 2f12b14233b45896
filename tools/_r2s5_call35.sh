for c in 1 5; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/s5c35_bench_cfg$c.json 2> gpurun_out/s5c35_bench_cfg$c.err; done
XCB_FORK_PREP=0 timeout 400 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu > gpurun_out/s5c35_bench_cfg1_off.json 2> gpurun_out/s5c35_bench_cfg1_off.err
timeout 400 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu > gpurun_out/s5c35_bench_cfg1b.json 2> gpurun_out/s5c35_bench_cfg1b.err
timeout 600 python tools/host_overhead.py > gpurun_out/s5c35_host_overhead.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s5c35_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c35_gpu_tests.log
