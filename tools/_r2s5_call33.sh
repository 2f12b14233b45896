timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s5c33_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c33_gpu_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s5c33_bench_cfg5.json 2> gpurun_out/s5c33_bench_cfg5.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5c33_smoke.log 2>&1
