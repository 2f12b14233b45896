for c in 1 2; do timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu > gpurun_out/s5c29_bench_cfg$c.json 2> gpurun_out/s5c29_bench_cfg$c.err; done
