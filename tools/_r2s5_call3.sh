timeout 900 python -m pytest tests/test_gpu_cpair.py -x -q > gpurun_out/s5c3_cpair_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c3_cpair_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_detect.py tests/test_contour.py -x -q -k "scatter or config2 or full_size_sampled or detect or contour or smooth or config4" > gpurun_out/s5c3_scatter_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c3_scatter_tests.log
timeout 400 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/s5c3_bench_cfg2_pre.json 2> gpurun_out/s5c3_bench_cfg2_pre.err
mkdir -p /tmp/reps; rm -f /tmp/reps/*
N="ncu --set full --clock-control none --import-source on -f"
timeout 600 $N -k regex:"premul|mac|inv_out|k_prep" -c 4 -o /tmp/reps/cfg2 python tools/profile_case.py xconv 2 > /dev/null 2>&1
cp profiles/ncu_kernel_stats.json gpurun_out/s5c3_ncu_kernel_stats.json
python tools/ncu_stats.py gpurun_out/s5c3_ncu_kernel_stats.json 2:/tmp/reps/cfg2.ncu-rep > /dev/null 2> gpurun_out/s5c3_stats.err
ncu -i /tmp/reps/cfg2.ncu-rep --page raw --csv > /tmp/reps/cfg2.raw.csv 2>/dev/null; python tools/ncu_summary.py /tmp/reps/cfg2.raw.csv > gpurun_out/s5c3_ncu_full_cfg2.txt
cp gpurun_out/s5c3_ncu_kernel_stats.json profiles/ncu_kernel_stats.json
timeout 400 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/s5c3_bench_cfg2.json 2> gpurun_out/s5c3_bench_cfg2.err
timeout 400 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu > gpurun_out/s5c3_bench_cfg4.json 2> gpurun_out/s5c3_bench_cfg4.err
