timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_cpp_shim.py -x -q > gpurun_out/c3_multi.log 2>&1
echo rc=$? >> gpurun_out/c3_multi.log
timeout 1200 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_fullsize.py > gpurun_out/c3_gpu_all.log 2>&1
echo rc=$? >> gpurun_out/c3_gpu_all.log
python tools/bench_configs.py 4 > gpurun_out/c3_cfg4.jsonl 2>&1
