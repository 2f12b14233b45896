set -x
timeout 300 python -m pytest tests/test_gpu_anglemax_tc.py -x -q > gpurun_out/r2c9_tc.log 2>&1; echo rc=$? >> gpurun_out/r2c9_tc.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py -x -q -k "anglemax or config3 or spatial" > gpurun_out/r2c9_am.log 2>&1; echo rc=$? >> gpurun_out/r2c9_am.log
XCB_ANGLE_TC=0 timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu > gpurun_out/r2c9_bench_cfg3_cuda.json 2> gpurun_out/r2c9_bench_cfg3_cuda.err
timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu > gpurun_out/r2c9_bench_cfg3.json 2> gpurun_out/r2c9_bench_cfg3.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"anglemax_tc" -c 1 -o /tmp/am_tc python tools/profile_case.py anglemax 3 > gpurun_out/r2c9_ncu.log 2>&1
ncu -i /tmp/am_tc.ncu-rep --page raw --csv > /tmp/am_tc.csv 2>/dev/null; python tools/ncu_summary.py /tmp/am_tc.csv > gpurun_out/r2c9_ncu_tc.txt
ncu -i /tmp/am_tc.ncu-rep --page source --csv --print-source sass > /tmp/am_src.csv 2>/dev/null; python tools/ncu_hot.py /tmp/am_src.csv 40 > gpurun_out/r2c9_tc_hot.txt 2>&1
