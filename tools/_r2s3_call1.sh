nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s3c1_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3c1_smoke.log 2>&1; echo rc=$? >> gpurun_out/s3c1_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3c1_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s3c1_gpu_tests.log
for c in 5 1 2 3 4; do timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/s3c1_bench_cfg$c.json 2> gpurun_out/s3c1_bench_cfg$c.err; done
timeout 400 python bench.py > gpurun_out/s3c1_bench_default.json 2> gpurun_out/s3c1_bench_default.err
