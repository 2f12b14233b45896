set -x
timeout 900 python -m pytest tests/test_gpu_fft.py tests/test_gpu_smooth_pack.py -x -q > gpurun_out/r2c8_fft.log 2>&1; echo rc=$? >> gpurun_out/r2c8_fft.log
mkdir -p /tmp/reps
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:"inv_corr|inv_steer|rows_fwd_ilv|cols_fwd_ilv|k_prep" -c 5 -o /tmp/reps/cfg5 python tools/profile_case.py xcorr 5 > gpurun_out/r2c8_ncu5.log 2>&1
timeout 600 $N -k regex:"premul|mac|inv_out|k_prep" -c 4 -o /tmp/reps/cfg2 python tools/profile_case.py xconv 2 > gpurun_out/r2c8_ncu2.log 2>&1
timeout 600 $N -k regex:"premul|mac|inv_out|smooth|absmax|k_prep" -c 7 -o /tmp/reps/cfg4 python tools/profile_case.py smooth 4 > gpurun_out/r2c8_ncu4.log 2>&1
timeout 900 $N -k regex:"inv_corr|inv_planes|anglemax|rows_fwd_ilv|cols_fwd_ilv" -c 5 -o /tmp/reps/cfg3 python tools/profile_case.py anglemax 3 > gpurun_out/r2c8_ncu3.log 2>&1
timeout 600 $N -k regex:"." -c 12 -o /tmp/reps/cfg1 python tools/profile_case.py xcorr 1 > gpurun_out/r2c8_ncu1.log 2>&1
python tools/ncu_stats.py gpurun_out/r2c8_ncu_kernel_stats.json 5:/tmp/reps/cfg5.ncu-rep 2:/tmp/reps/cfg2.ncu-rep 4:/tmp/reps/cfg4.ncu-rep 3:/tmp/reps/cfg3.ncu-rep 1:/tmp/reps/cfg1.ncu-rep > /dev/null 2> gpurun_out/r2c8_stats.err
for c in 5 2 4 3 1; do ncu -i /tmp/reps/cfg$c.ncu-rep --page raw --csv > /tmp/reps/cfg$c.raw.csv 2>/dev/null; python tools/ncu_summary.py /tmp/reps/cfg$c.raw.csv > gpurun_out/r2c8_ncu_full_cfg$c.txt; done
cp gpurun_out/r2c8_ncu_kernel_stats.json profiles/ncu_kernel_stats.json
for c in 5 2 3 4 1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2c8_bench_cfg$c.json 2> gpurun_out/r2c8_bench_cfg$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c8_launches_cfg5.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
du -sh gpurun_out
