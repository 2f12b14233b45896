timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s5c28_bench_cfg5.json 2> gpurun_out/s5c28_bench_cfg5.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s5c28_bench_reference.json 2> gpurun_out/s5c28_bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5c28_launches_cfg5.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5c28_launches_cfg2.csv python bench.py --config 2 --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5c28_launches_cfg1.csv python bench.py --config 1 --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
mkdir -p /tmp/reps; rm -f /tmp/reps/*
N="ncu --set full --clock-control none --import-source on -f"
timeout 900 $N -k regex:"inv_corr|inv_steer" -c 4 -o /tmp/reps/cfg5 python tools/profile_case.py xcorr 5 1 > /dev/null 2>&1
ncu -i /tmp/reps/cfg5.ncu-rep --page raw --csv > /tmp/reps/cfg5.raw.csv 2>/dev/null; python tools/ncu_summary.py /tmp/reps/cfg5.raw.csv > gpurun_out/s5c28_ncu_full_cfg5.txt
cp profiles/ncu_kernel_stats.json gpurun_out/s5c28_ncu_kernel_stats.json
python tools/ncu_stats.py gpurun_out/s5c28_ncu_kernel_stats.json 5:/tmp/reps/cfg5.ncu-rep > /dev/null 2> gpurun_out/s5c28_stats.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5c28_smoke.log 2>&1
