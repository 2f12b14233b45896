set -x
timeout 1500 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/r2c21_gpu_all.log 2>&1; echo rc=$? >> gpurun_out/r2c21_gpu_all.log
mkdir -p /tmp/reps21; rm -f /tmp/reps21/*
N="ncu --set full --clock-control none --import-source on -f"
timeout 600 $N -k regex:"premul|mac|inv_out|k_prep" -c 4 -o /tmp/reps21/cfg2 python tools/profile_case.py xconv 2 > /dev/null 2>&1
timeout 900 $N -k regex:"inv_corr|inv_planes|anglemax|rows_fwd_ilv|cols_fwd_ilv" -c 5 -o /tmp/reps21/cfg3 python tools/profile_case.py anglemax 3 > /dev/null 2>&1
cp profiles/ncu_kernel_stats.json gpurun_out/r2c21_ncu_kernel_stats.json
python tools/ncu_stats.py gpurun_out/r2c21_ncu_kernel_stats.json 2:/tmp/reps21/cfg2.ncu-rep 3:/tmp/reps21/cfg3.ncu-rep > /dev/null 2> gpurun_out/r2c21_stats.err
for c in 2 3; do ncu -i /tmp/reps21/cfg$c.ncu-rep --page raw --csv > /tmp/reps21/cfg$c.raw.csv 2>/dev/null; python tools/ncu_summary.py /tmp/reps21/cfg$c.raw.csv > gpurun_out/r2c21_ncu_full_cfg$c.txt; done
cp gpurun_out/r2c21_ncu_kernel_stats.json profiles/ncu_kernel_stats.json
for c in 5 2 3 4 1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2c21_bench_cfg$c.json 2> gpurun_out/r2c21_bench_cfg$c.err; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2c21_ref_cfg5.json 2> gpurun_out/r2c21_ref_cfg5.err
