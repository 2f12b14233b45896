set -x
timeout 600 python -m pytest tests/test_gpu_smooth_pack.py tests/test_gpu_sharded.py -x -q > gpurun_out/r2c7_pack.log 2>&1; echo rc=$? >> gpurun_out/r2c7_pack.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2c7_gpu_all.log 2>&1; echo rc=$? >> gpurun_out/r2c7_gpu_all.log
mkdir -p /tmp/reps
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:"inv_corr|inv_steer|rows_fwd_ilv|cols_fwd_ilv|k_prep" -c 5 -o /tmp/reps/cfg5 python tools/profile_case.py xcorr 5 > gpurun_out/r2c7_ncu5.log 2>&1
timeout 600 $N -k regex:"premul|mac|inv_out|k_prep" -c 4 -o /tmp/reps/cfg2 python tools/profile_case.py xconv 2 > gpurun_out/r2c7_ncu2.log 2>&1
timeout 600 $N -k regex:"premul|mac|inv_out|smooth|absmax|k_prep" -c 7 -o /tmp/reps/cfg4 python tools/profile_case.py smooth 4 > gpurun_out/r2c7_ncu4.log 2>&1
timeout 900 $N -k regex:"inv_corr|inv_planes|anglemax|rows_fwd_ilv|cols_fwd_ilv" -c 5 -o /tmp/reps/cfg3 python tools/profile_case.py anglemax 3 > gpurun_out/r2c7_ncu3.log 2>&1
python tools/ncu_stats.py gpurun_out/r2c7_ncu_kernel_stats.json 5:/tmp/reps/cfg5.ncu-rep 2:/tmp/reps/cfg2.ncu-rep 4:/tmp/reps/cfg4.ncu-rep 3:/tmp/reps/cfg3.ncu-rep > /dev/null 2> gpurun_out/r2c7_stats.err
for c in 5 2 4 3; do ncu -i /tmp/reps/cfg$c.ncu-rep --page raw --csv > /tmp/reps/cfg$c.raw.csv 2>/dev/null; python tools/ncu_summary.py /tmp/reps/cfg$c.raw.csv > gpurun_out/r2c7_ncu_full_cfg$c.txt; done
ncu -i /tmp/reps/cfg2.ncu-rep --page source --csv --print-source sass -k regex:premul > /tmp/reps/s1src.csv 2>/dev/null; python tools/ncu_hot.py /tmp/reps/s1src.csv 30 > gpurun_out/r2c7_s1_hot.txt 2>&1
cp /tmp/reps/cfg2.ncu-rep gpurun_out/r2c7_full_cfg2.ncu-rep
du -sh gpurun_out
