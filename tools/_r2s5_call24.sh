timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s5c24_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c24_gpu_tests.log
for c in 1 2 4 3; do timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu > gpurun_out/s5c24_bench_cfg$c.json 2> gpurun_out/s5c24_bench_cfg$c.err; done
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s5c24_bench_cfg5.json 2> gpurun_out/s5c24_bench_cfg5.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5c24_smoke.log 2>&1
