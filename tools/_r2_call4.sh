set -x
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/r2c4_gpu_all.log 2>&1; echo rc=$? >> gpurun_out/r2c4_gpu_all.log
timeout 600 python tools/ab_kernels.py --case "xconv 2" --regex "premul|mac|inv_out" cur s1p > gpurun_out/r2c4_ab_cfg2.txt 2>&1
for c in 2 4 1; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/r2c4_bench_cfg$c.json 2> gpurun_out/r2c4_bench_cfg$c.err; done
