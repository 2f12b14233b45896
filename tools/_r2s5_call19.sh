timeout 600 python tools/e2e_breakdown.py > gpurun_out/s5c19_e2e.txt 2>&1
