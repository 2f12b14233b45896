set -x
timeout 600 python -m pytest tests/test_gpu_smooth_pack.py -x -q > gpurun_out/r2c6_pack.log 2>&1; echo rc=$? >> gpurun_out/r2c6_pack.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2c6_gpu_all.log 2>&1; echo rc=$? >> gpurun_out/r2c6_gpu_all.log
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:"inv_corr|inv_steer|rows_fwd_ilv|cols_fwd_ilv|k_prep" -c 5 -o gpurun_out/r2c6_full_cfg5 python tools/profile_case.py xcorr 5 > gpurun_out/r2c6_ncu5.log 2>&1
timeout 600 $N -k regex:"premul|mac|inv_out|k_prep" -c 4 -o gpurun_out/r2c6_full_cfg2 python tools/profile_case.py xconv 2 > gpurun_out/r2c6_ncu2.log 2>&1
timeout 600 $N -k regex:"premul|mac|inv_out|smooth|absmax|k_prep" -c 7 -o gpurun_out/r2c6_full_cfg4 python tools/profile_case.py smooth 4 > gpurun_out/r2c6_ncu4.log 2>&1
timeout 900 $N -k regex:"inv_corr|inv_planes|anglemax|rows_fwd_ilv|cols_fwd_ilv" -c 5 -o gpurun_out/r2c6_full_cfg3 python tools/profile_case.py anglemax 3 > gpurun_out/r2c6_ncu3.log 2>&1
for c in 2 4; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/r2c6_bench_cfg$c.json 2> gpurun_out/r2c6_bench_cfg$c.err; done
