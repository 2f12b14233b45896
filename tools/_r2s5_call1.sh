timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s5c1_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c1_gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/s5c1_bench_default.json 2> gpurun_out/s5c1_bench_default.err
for c in 2 4 3 1; do timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/s5c1_bench_cfg$c.json 2> gpurun_out/s5c1_bench_cfg$c.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s5c1_bench_reference.json 2> gpurun_out/s5c1_bench_reference.err
nvidia-smi > gpurun_out/s5c1_smi.txt
