python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5c36_smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cpair.py tests/test_gpu_tiles.py -x -q > gpurun_out/s5c36_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c36_tests.log
timeout 400 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu > gpurun_out/s5c36_bench_cfg1.json 2> gpurun_out/s5c36_bench_cfg1.err
