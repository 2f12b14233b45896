timeout 600 python tools/host_overhead.py > gpurun_out/s5c34_host_overhead.txt 2>&1
