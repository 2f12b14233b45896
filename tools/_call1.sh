set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c1_build.log 2>&1
python tools/bench_configs.py 1 2 3 4 > gpurun_out/c1_configs.jsonl 2> gpurun_out/c1_configs.err
for m in "xconv 2" "smooth 4"; do
  set -- $m
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1_launch_$1_$2.csv python tools/profile_case.py $1 $2 > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"premul|mac|inv_out" -c 3 -o gpurun_out/c1_full_$1_$2 python tools/profile_case.py $1 $2 > gpurun_out/c1_ncu_$1_$2.log 2>&1
done
ls -la gpurun_out
