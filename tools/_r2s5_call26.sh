mkdir -p /tmp/reps; rm -f /tmp/reps/*
N="ncu --set full --clock-control none --import-source on -f"
timeout 600 $N -k regex:"inv_corr|inv_steer|rows_fwd_ilv|cols_fwd_ilv|k_prep" -c 5 -o /tmp/reps/cfg1 python tools/profile_case.py xcorr 1 > /dev/null 2>&1
cp profiles/ncu_kernel_stats.json gpurun_out/s5c26_ncu_kernel_stats.json
python tools/ncu_stats.py gpurun_out/s5c26_ncu_kernel_stats.json 1:/tmp/reps/cfg1.ncu-rep > /dev/null 2> gpurun_out/s5c26_stats.err
ncu -i /tmp/reps/cfg1.ncu-rep --page raw --csv > /tmp/reps/cfg1.raw.csv 2>/dev/null; python tools/ncu_summary.py /tmp/reps/cfg1.raw.csv > gpurun_out/s5c26_ncu_full_cfg1.txt
cp gpurun_out/s5c26_ncu_kernel_stats.json profiles/ncu_kernel_stats.json
timeout 400 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu > gpurun_out/s5c26_bench_cfg1.json 2> gpurun_out/s5c26_bench_cfg1.err
