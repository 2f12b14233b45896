set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2c1_host.txt; nproc >> gpurun_out/r2c1_host.txt; lscpu | grep "Model name" >> gpurun_out/r2c1_host.txt
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2c1_gpu_all.log 2>&1; echo rc=$? >> gpurun_out/r2c1_gpu_all.log
for c in 5 2 3 4 1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2c1_bench_cfg$c.json 2> gpurun_out/r2c1_bench_cfg$c.err; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2c1_ref_cfg5.json 2> gpurun_out/r2c1_ref_cfg5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c1_launches_cfg5.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2c1_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"inv_steer|inv_corr" -c 2 -o gpurun_out/r2c1_full_cfg5 python tools/profile_case.py xcorr 5 > gpurun_out/r2c1_ncu_full.log 2>&1
for m in "xconv 2" "smooth 4"; do set -- $m
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"premul|mac|inv_out" -c 3 -o gpurun_out/r2c1_full_$1_$2 python tools/profile_case.py $1 $2 > gpurun_out/r2c1_ncu_$1_$2.log 2>&1
done
ls -la gpurun_out
