timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/c5_multi.log 2>&1; echo rc=$? >> gpurun_out/c5_multi.log
for c in 5 2 3 4 1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/c5_bench_cfg$c.json 2> gpurun_out/c5_bench_cfg$c.err; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/c5_ref_cfg5.json 2> gpurun_out/c5_ref_cfg5.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --shard bands > gpurun_out/c5_tr_bands.json 2> gpurun_out/c5_tr_bands.err
