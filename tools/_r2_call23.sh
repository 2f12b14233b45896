timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py tests/test_gpu_ref.py tests/test_cpp_shim.py tests/test_gpu_guards.py tests/test_detect.py -x -q > gpurun_out/r2c23_par.log 2>&1; echo rc=$? >> gpurun_out/r2c23_par.log
timeout 300 python bench.py --config 1 --steps 50 --warmup 5 --no-cpu > gpurun_out/r2c23_bench_cfg1.json 2> gpurun_out/r2c23_bench_cfg1.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c23_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2c23_smoke.log
