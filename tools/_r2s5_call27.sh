for c in 1 2 4; do timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu > gpurun_out/s5c27_bench_cfg$c.json 2> gpurun_out/s5c27_bench_cfg$c.err; done
for c in 1 2 4; do XCB_PDL=0 timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu > gpurun_out/s5c27_bench_cfg${c}_off.json 2> gpurun_out/s5c27_bench_cfg${c}_off.err; done
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s5c27_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c27_gpu_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/s5c27_bench_cfg5.json 2> gpurun_out/s5c27_bench_cfg5.err
timeout 400 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu > gpurun_out/s5c27_bench_cfg3.json 2> gpurun_out/s5c27_bench_cfg3.err
