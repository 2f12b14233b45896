nproc > gpurun_out/c2_host.txt; free -g >> gpurun_out/c2_host.txt; lscpu | grep "Model name" >> gpurun_out/c2_host.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -v --durations=0 > gpurun_out/c2_fullsize.log 2>&1
echo rc=$? >> gpurun_out/c2_fullsize.log
