timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s5c20_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s5c20_gpu_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s5c20_bench_cfg5.json 2> gpurun_out/s5c20_bench_cfg5.err
for c in 2 4 3 1; do timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu > gpurun_out/s5c20_bench_cfg$c.json 2> gpurun_out/s5c20_bench_cfg$c.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s5c20_bench_reference.json 2> gpurun_out/s5c20_bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5c20_launches_cfg5.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5c20_launches_cfg2.csv python bench.py --config 2 --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5c20_smoke.log 2>&1
