set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2c2_gpu_all.log 2>&1; echo rc=$? >> gpurun_out/r2c2_gpu_all.log
timeout 600 python tools/ab_kernels.py --case "xconv 2" --regex "premul|mac|inv_out" base dk1 > gpurun_out/r2c2_ab_cfg2.txt 2>&1
timeout 600 python tools/ab_kernels.py --case "smooth 4" --regex "premul|mac|inv_out" base dk1 > gpurun_out/r2c2_ab_cfg4.txt 2>&1
timeout 600 python tools/ab_kernels.py --case "xcorr 5" --regex "ilv" base dk1 > gpurun_out/r2c2_ab_cfg5.txt 2>&1
for t in memcheck racecheck synccheck; do for c in "xconv 2" "smooth 4" "xcorr 1" "anglemax 3"; do set -- $c
timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/profile_case.py $1 $2 > gpurun_out/r2c2_san_${t}_$1_$2.log 2>&1; echo rc=$? >> gpurun_out/r2c2_san_${t}_$1_$2.log
done; done
timeout 1200 compute-sanitizer --tool memcheck --print-limit 50 python tools/profile_case.py xcorr 5 > gpurun_out/r2c2_san_memcheck_xcorr_5.log 2>&1; echo rc=$? >> gpurun_out/r2c2_san_memcheck_xcorr_5.log
for c in 2 4 5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/r2c2_bench_cfg$c.json 2> gpurun_out/r2c2_bench_cfg$c.err; done
