timeout 300 python -m pytest tests/test_gpu_anglemax_tc.py -x -q > gpurun_out/r2c19_tc.log 2>&1; echo rc=$? >> gpurun_out/r2c19_tc.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:anglemax_tc -c 2 --csv python tools/profile_case.py anglemax 3 2>/dev/null | grep anglemax_tc | tail -1 | awk -F'","' '{print $NF}' > gpurun_out/r2c19_time.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py tests/test_gpu_guards.py -x -q -k "anglemax or config3 or spatial or guard" > gpurun_out/r2c19_am.log 2>&1; echo rc=$? >> gpurun_out/r2c19_am.log
timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu > gpurun_out/r2c19_bench_cfg3.json 2> gpurun_out/r2c19_bench_cfg3.err
