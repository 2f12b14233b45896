timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s5c12_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c12_gpu_tests.log
for c in 1 2 3 4; do timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu > gpurun_out/s5c12_bench_cfg$c.json 2> gpurun_out/s5c12_bench_cfg$c.err; done
