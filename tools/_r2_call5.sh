set -x
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/r2c5_gpu_all.log 2>&1; echo rc=$? >> gpurun_out/r2c5_gpu_all.log
XCB_PACK=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_ref.py -x -q -k "smooth or config4" > gpurun_out/r2c5_nopack.log 2>&1; echo rc=$? >> gpurun_out/r2c5_nopack.log
timeout 600 python tools/ab_kernels.py --case "smooth 4" --regex "premul|mac|inv_out|smooth|absmax" s1p pack > gpurun_out/r2c5_ab_cfg4.txt 2>&1
timeout 600 python tools/ab_kernels.py --case "xconv 2" --regex "premul|mac|inv_out" cur s1p > gpurun_out/r2c5_ab_cfg2.txt 2>&1
for c in 4 2; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/r2c5_bench_cfg$c.json 2> gpurun_out/r2c5_bench_cfg$c.err; done
XCB_PACK=0 timeout 600 python bench.py --config 4 --steps 20 --warmup 5 --no-cpu > gpurun_out/r2c5_bench_cfg4_nopack.json 2> gpurun_out/r2c5_bench_cfg4_nopack.err
