set -x
XCB_TC_VARIANT=3 timeout 300 python -m pytest tests/test_gpu_anglemax_tc.py -x -q > gpurun_out/r2c14_tc_v3.log 2>&1; echo rc=$? >> gpurun_out/r2c14_tc_v3.log
for v in 2 3; do XCB_TC_VARIANT=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:anglemax_tc -c 2 --csv python tools/profile_case.py anglemax 3 2>/dev/null | grep anglemax_tc | tail -1 | awk -F'","' -v v=$v '{print "v" v " " $NF}' >> gpurun_out/r2c14_times.txt; done
XCB_TC_VARIANT=3 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"anglemax_tc" -c 1 -o /tmp/am16 python tools/profile_case.py anglemax 3 > /dev/null 2>&1
ncu -i /tmp/am16.ncu-rep --page raw --csv > /tmp/am16.csv 2>/dev/null; python tools/ncu_summary.py /tmp/am16.csv > gpurun_out/r2c14_ncu16.txt
grep -o '"sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed","[^"]*","[^"]*"' /tmp/am16.csv >> gpurun_out/r2c14_ncu16.txt
ncu -i /tmp/am16.ncu-rep --page source --csv --print-source sass > /tmp/am16src.csv 2>/dev/null; python tools/ncu_hot.py /tmp/am16src.csv 30 > gpurun_out/r2c14_hot16.txt 2>&1
